# round 2: full GPU suite with the stale-register gathers, K1 A/B (zero-filled vs
# stale), end-to-end breakdown, quick bench (no configs 3/4)
python -m pytest tests -m gpu -q -x > gpurun_out/t4.log 2>&1; tail -3 gpurun_out/t4.log
for lib in libcsemb_cuda_zero.so libcsemb_cuda.so libcsemb_cuda_zero.so libcsemb_cuda.so; do
  echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm --widths 80,40,10 --L 20 2>&1 | grep K1
done > gpurun_out/stale_ab.log 2>&1; cat gpurun_out/stale_ab.log
python tools/e2e_breakdown.py > gpurun_out/e2e_bd2.log 2>&1; tail -2 gpurun_out/e2e_bd2.log
python bench.py --skip-configs34 --skip-cpu > gpurun_out/b4.json 2> gpurun_out/b4.log; grep "\[bench\]" gpurun_out/b4.log
