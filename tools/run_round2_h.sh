# session-2 baseline check on a fresh box: GPU suite, smoke, bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/h_smoke.log 2>&1; tail -2 gpurun_out/h_smoke.log
timeout 900 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc=$?"
head -c 600 gpurun_out/h_bench.json
