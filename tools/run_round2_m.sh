# K1_UNCOND (no per-entry predicates / zero-fill) x TRIM x EARLY
for rep in 1 2; do
for v in "" _u _ut _ute; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80,40 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_u.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/m_parity_u.log 2>&1; echo "parity u rc=$?"; tail -3 gpurun_out/m_parity_u.log
