python -m pytest tests/test_gpu_parity.py tests/test_reference_suite.py tests/test_gpu_scale.py -m gpu -q -s -k "DeviceBuild or device_list or graph_survives or nccl or reference_suite or config3" > gpurun_out/t3.log 2>&1; tail -5 gpurun_out/t3.log
python tools/e2e_breakdown.py > gpurun_out/e2e_bd.log 2>&1; tail -3 gpurun_out/e2e_bd.log
for v in 3 4 5; do for lib in libcsemb_cuda.so libcsemb_cuda_wide.so; do
  [ $lib = libcsemb_cuda.so ] && [ $v != 3 ] && continue
  echo "== $lib target $v"; CSEMB_TARGET_VPL=$v CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm --widths 80,40,96 --L 20 2>&1 | grep K1
done; done > gpurun_out/wide.log 2>&1; cat gpurun_out/wide.log
