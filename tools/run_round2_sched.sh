# device-built schedule order vs the host path: build time (trace build) and K1 time / e2e (must be identical)
for h in "" 1; do
  echo "== CSEMB_SCHED_HOST=$h"
  CSEMB_SCHED_HOST=$h CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_trace.so timeout 600 python tools/e2e_breakdown.py 2>&1 | grep -v Warn | tail -4
  CSEMB_SCHED_HOST=$h timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80,10 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/sched_pytest.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/sched_pytest.log
