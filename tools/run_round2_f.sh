# fp64 K1 with fused multiply-add (K1_FMA64 build) vs the strict separately-rounded form
for lib in libcsemb_cuda.so libcsemb_cuda_fma.so libcsemb_cuda.so libcsemb_cuda_fma.so; do
  echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f64 --graphs sbm --widths 80,40 --L 20 2>&1 | grep K1
done
for lib in libcsemb_cuda.so libcsemb_cuda_fma.so; do
  echo "== sustained bench f64 $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib python bench.py --skip-fp32 --skip-e2e --skip-downstream --skip-cpu --skip-configs34 --skip-builders 2>&1 | grep "\[bench\] f64"
done
