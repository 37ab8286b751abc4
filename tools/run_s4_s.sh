# session 4: window length cap sweep under the column rule (config 4 / 3 fp32, full L)
for ml in 65536 16384 32768 131072 262144 65536; do
  CSEMB_HEAVY_WINDOW_MAXLEN=$ml timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/maxlen=$ml /"
done
