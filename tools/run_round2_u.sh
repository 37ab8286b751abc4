# narrow column shards (d=10): K1 vs its floor, and the epilogue share (K1_ABLATE builds: 1 no stream loads, 4 no stores, 5 both)
for v in "" _ab1 _ab4 _ab5; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm --widths 10,20 2>&1 | grep K1
done
