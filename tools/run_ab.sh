# A/B of two library builds on the sustained, power-capped bench (A, B interleaved twice)
A=${A:-libcsemb_cuda_nopf.so}; B=${B:-libcsemb_cuda.so}
for lib in $A $B $A $B; do
  echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python bench.py --skip-cpu --skip-e2e --skip-downstream 2>&1 | grep "\[bench\]"
done
