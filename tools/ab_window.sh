set -x
for w in 0 40 20 80; do
  CSEMB_HEAVY_WINDOW_MB=$w timeout 300 python tools/bench_configs.py --configs 4,3 --dtype f32,f64 --reps 2 2>&1 | sed "s/^/w=$w /"
done
