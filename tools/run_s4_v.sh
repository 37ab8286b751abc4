# session 4: fixed chunks of the hottest rows swept first (their own first-column order), windowed pieces after
for ff in 0 1 0 1; do
  if [ $ff = 1 ]; then export CSEMB_WINDOW_FIXED_FIRST=1; else unset CSEMB_WINDOW_FIXED_FIRST; fi
  timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/fixed_first=$ff /"
done
