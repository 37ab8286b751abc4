# split exchange + value-free GPU tests; K1 with the value-free branch compiled in (default off) vs compiled out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or ValueFree or nccl_driver or emulated" > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/q_tests.log
for rep in 1 2; do
for v in "" _novf; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80,40 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
