# K1 ablations against the gather floor (sbm, d=80)
for v in "" _ab1 _ab4 _ab5; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80 2>&1 | grep K1
done
