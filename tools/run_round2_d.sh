# narrow column shards: lanes per row (CSEMB_TARGET_VPL 1 = one 16-byte vector per lane,
# contiguous row segments per load instruction) vs the default 3 vectors per lane
for v in 3 1 2 3 1; do
  echo "== target vpl $v"; CSEMB_TARGET_VPL=$v CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_v1.so timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm --widths 10,20,40 --L 20 2>&1 | grep K1
done > gpurun_out/vpl_narrow.log 2>&1; cat gpurun_out/vpl_narrow.log
