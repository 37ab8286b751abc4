# session 4: staged entry batches for narrow groups (column-shard widths)
export CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_narrow.so
CSEMB_K1_STAGE_NARROW=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "widths or Config1 or EdgeCases" 2>&1 | tail -2
for rep in 1 2; do
  echo "== base"; timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm --widths 40,20,10 --L 20 2>&1 | grep K1
  echo "== narrow staged"; CSEMB_K1_STAGE_NARROW=1 timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm --widths 40,20,10 --L 20 2>&1 | grep K1
done
