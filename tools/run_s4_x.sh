# session 4: staged entry batches in fp64 on the skewed configs (full L, sustained)
for m in 0 3 0 3; do
  CSEMB_K1_TMA=$m timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f64 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/f64 tma=$m /"
done
