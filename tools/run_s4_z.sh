# session 4: epilogue L2 prefetch (fp64) on / off under the sustained, power-capped bench
for lib in libcsemb_cuda.so libcsemb_cuda_nopf.so libcsemb_cuda.so libcsemb_cuda_nopf.so; do
  echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 400 python bench.py --skip-cpu --skip-e2e --skip-downstream --skip-configs34 --skip-builders 2>&1 | grep "\[bench\] f64"
done
