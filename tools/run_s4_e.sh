# session 4: heavy-row chunks cut at L2-sized column windows, equal pieces, bucketed by length inside each window
for w in 0 32 48 64 96 160; do
  CSEMB_HEAVY_WINDOW_MB=$w timeout 400 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/window=$w MB /"
done
