# session 4: window width in columns (fp32 / fp64), config 4 and 3
for w in 131072 174762 196608 262144 0 174762 131072; do
  if [ $w = 0 ]; then export CSEMB_HEAVY_WINDOW_MB=0; else unset CSEMB_HEAVY_WINDOW_MB; export CSEMB_WINDOW_COLS_F32=$w; fi
  timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"dtype": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - - | sed "s/^/wcols32=$w /"
done
unset CSEMB_HEAVY_WINDOW_MB
for w in 65536 87381 131072 43690; do
  CSEMB_WINDOW_COLS_F64=$w timeout 600 python tools/bench_configs.py --configs 4 --dtype f64 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"dtype": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - - | sed "s/^/wcols64=$w /"
done
