# per-kernel time split of config 4 (heavy-row chunks / light rows / combine) from an ncu launch list
C="python tools/bench_configs.py --configs 4 --dtype f32 --reps 0"
$C > gpurun_out/c4plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/c4_launches.csv $C > /dev/null 2>&1
echo rc=$?
