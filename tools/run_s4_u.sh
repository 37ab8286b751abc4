# session 4: entries-per-window requirement sweep (config 4 / 3 fp32, full L)
for per in 20 10 14 30 40 20; do
  CSEMB_WINDOW_MIN_PER=$per timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/per=$per /"
done
