# session 4: width-independent window rule (2^17 / 2^16 columns) -- invariance test, configs 3/4 vs windows off, full suite
timeout 900 python -m pytest tests/test_gpu_scale.py -m gpu -x -q -k windowed_heavy_rows 2>&1 | tail -3
for w in auto 0 auto 0; do
  if [ $w = auto ]; then unset CSEMB_HEAVY_WINDOW_MB; else export CSEMB_HEAVY_WINDOW_MB=$w; fi
  timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32,f64 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"dtype": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - - | sed "s/^/window=$w /"
done
unset CSEMB_HEAVY_WINDOW_MB
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_o_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_o_pytest.log
