timeout 900 python bench.py > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err; echo "bench rc=$?"
tail -12 gpurun_out/o_bench.err
