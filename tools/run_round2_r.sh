# split exchange, one rank's share: config 5 at full scale (rank 0 of 8) and a config-2-sized graph (rank 0 of 8, f64)
timeout 900 python tools/bench_config5_rank.py --split --out gpurun_out/r_config5_split.json > gpurun_out/r_c5.log 2>&1; echo "c5 rc=$?"; tail -2 gpurun_out/r_c5.log
timeout 600 python tools/bench_config5_rank.py --split --n 1000000 --block 10000 --gpus 8 --d 80 --dtype f64 --steps 10 --out gpurun_out/r_config2_split.json > gpurun_out/r_c2.log 2>&1; echo "c2 rc=$?"; tail -2 gpurun_out/r_c2.log
