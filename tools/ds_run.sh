timeout 600 python -m pytest tests/test_gpu_downstream.py -q -x 2>&1 | tail -3
P=18.56
timeout 600 python tools/bench_downstream.py --fp64-peak $P --out gpurun_out/downstream.json 2>&1 | tail -2
timeout 300 python tools/bench_downstream.py --fp64-peak $P --max-iters 6 --cpu 0 > gpurun_out/ds_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_km|k_pair|k_modul|k_chunk|k_sum|k_argmax|k_sqnorm" --csv --log-file gpurun_out/ds_launches.csv python tools/bench_downstream.py --fp64-peak $P --max-iters 6 --cpu 0 > gpurun_out/ds_ncu.log 2>&1; echo ncu_rc=$?
