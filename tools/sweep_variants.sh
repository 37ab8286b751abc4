# K1 build variants on config-2-sized graphs (K1_MIN_BLOCKS / GATHER_MODE builds x CSEMB_TARGET_VPL)
for lib in ${LIBS:-libcsemb_cuda.so libcsemb_cuda_mb4.so libcsemb_cuda_g1.so libcsemb_cuda_g2.so}; do
 for tv in ${TVS:-5 3}; do
   echo "== $lib tv=$tv"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib CSEMB_TARGET_VPL=$tv timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs ${GRAPHS:-band,sbm} 2>&1 | grep K1
 done
done
