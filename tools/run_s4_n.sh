# session 4: automatic column windows for moderately heavy rows -- full suite, configs 3/4 in both dtypes vs windows off
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_n_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_n_pytest.log
for w in auto 0 auto 0; do
  if [ $w = auto ]; then unset CSEMB_HEAVY_WINDOW_MB; else export CSEMB_HEAVY_WINDOW_MB=$w; fi
  timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32,f64 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"dtype": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - - | sed "s/^/window=$w /"
done
