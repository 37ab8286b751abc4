# fp32 K1 depth A/B (2 vs 4 gathers in flight per lane), then the full GPU suite
for lib in libcsemb_cuda.so libcsemb_cuda_d4.so libcsemb_cuda.so libcsemb_cuda_d4.so; do
  echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f32 --graphs sbm,random --widths 80,96 --L 20 2>&1 | grep K1
done > gpurun_out/d4_ab.log 2>&1; cat gpurun_out/d4_ab.log
CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_d4.so timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*'
python -m pytest tests -m gpu -q > gpurun_out/t5.log 2>&1; tail -3 gpurun_out/t5.log
