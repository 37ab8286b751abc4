timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/up_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/up_pytest.log
timeout 600 python tools/upload_probe.py 2>&1 | tail -2
timeout 900 python bench.py --skip-cpu --skip-downstream --skip-configs34 --skip-builders > gpurun_out/up_bench.json 2> gpurun_out/up_bench.err; tail -3 gpurun_out/up_bench.err
