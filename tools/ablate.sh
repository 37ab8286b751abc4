# K1 ablation builds (timing only): 1 no stream loads, 2 local gathers, 4 no stores
for lib in libcsemb_cuda.so libcsemb_cuda_ab1.so libcsemb_cuda_ab2.so libcsemb_cuda_ab4.so libcsemb_cuda_ab3.so; do
  echo "== $lib"; CSEMB_K1_STAGED=0 CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm 2>&1 | grep K1
done
