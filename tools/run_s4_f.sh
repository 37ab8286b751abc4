# session 4: hot heavy rows cut at tiny column windows, swept window by window (L1 reuse of the gathered rows)
for cfg in "0 256" "64 256" "128 256" "256 256" "128 512" "256 128" "512 256"; do
  set -- $cfg
  CSEMB_HOT_ROWS=$1 CSEMB_HOT_WINDOW=$2 timeout 400 python tools/bench_configs.py --configs 4 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/hot=$1 window=$2 /"
done
