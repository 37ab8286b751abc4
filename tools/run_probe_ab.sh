# short-run K1 probe A/B of two library builds (config-2 SBM + uniform random graph)
A=${A:-libcsemb_cuda_nopf.so}; B=${B:-libcsemb_cuda.so}
for lib in $A $B $A $B; do
  echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs ${GRAPHS:-sbm,random} --widths ${WIDTHS:-80} --L 20 2>&1 | grep K1
done
