# K1 probe over several library builds, interleaved twice: LIBS="a.so b.so ..." WIDTHS=80,40
for rep in 1 2; do
  for lib in $LIBS; do
    echo "== $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs ${GRAPHS:-sbm} --widths ${WIDTHS:-80} --L 20 2>&1 | grep K1
  done
done
if [ -n "$BENCH" ]; then
  for rep in 1 2; do
    for lib in $LIBS; do
      echo "== bench $lib"; CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/$lib timeout 300 python bench.py --skip-cpu --skip-e2e --skip-downstream 2>&1 | grep "\[bench\] f"
    done
  done
fi
