# A/B of a runtime switch on one library: VAR=A vs VAR=B, short K1 probe and the sustained bench
VAR=${VAR:-CSEMB_K1_WIDE}; A=${A:-0}; B=${B:-1}
for v in $A $B $A $B; do
  echo "== $VAR=$v"; env $VAR=$v timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs ${GRAPHS:-sbm,random} --L 20 2>&1 | grep K1
done
if [ -n "$BENCH" ]; then
  for v in $A $B $A $B; do
    echo "== bench $VAR=$v"; env $VAR=$v timeout 300 python bench.py --skip-cpu --skip-e2e --skip-downstream 2>&1 | grep "\[bench\] f"
  done
fi
