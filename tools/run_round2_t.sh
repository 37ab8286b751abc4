# fp64 depth 2 on the shapes that spill at depth 4 (4- and 32-lane groups, exact peaks): spill-free, timed
for rep in 1 2; do
for v in "" _ns; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64 --graphs sbm,random --widths 20,24,120 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
