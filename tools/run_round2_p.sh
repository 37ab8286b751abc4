# fp32 gather depth 4 (K1_DEPTH_F32=4, spill-free on the d=80 shape now) vs shipped depth 2
for rep in 1 2; do
for v in "" _d4; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f32 --graphs sbm,random --widths 80,96,40 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
