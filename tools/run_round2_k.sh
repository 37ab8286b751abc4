# K1_EARLY (next row set's first batch loaded a row set ahead) x K1_TRIM
for rep in 1 2; do
for v in "" _early _trim _et; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80,40 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
