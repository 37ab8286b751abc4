# L2 fill-size hints: gathers (GATHER_MODE=3: L2::256B) and streamed loads (K1_STREAM_PF=1)
for rep in 1 2; do
for v in "" _g3 _spf _g3spf; do
  echo "== lib$v"
  CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda$v.so timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
