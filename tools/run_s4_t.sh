# session 4: demotion of locally-gathering rows -- variants, full suite, configs 3/4 unchanged?
timeout 1500 python -m pytest tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - -
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_t_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_t_pytest.log
