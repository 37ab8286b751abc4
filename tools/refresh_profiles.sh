# Round-end evidence refresh (one GPU): bench line, reference arm, ncu launch list,
# ncu --set full of K1 per dtype.  Each ncu pass runs only after its command
# exited 0 without ncu.  Summarise afterwards with: python tools/make_profiles.py <tag>
TAG=${TAG:-r2}
set -e
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-downstream --skip-configs34 --skip-builders > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --skip-downstream --skip-configs34 --skip-builders > gpurun_out/ncu_launch_$TAG.log 2>&1
for dt in f64 f32; do
  python tools/profile_k1.py --dtype $dt --L 6 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -f \
      -o gpurun_out/prof_${TAG}_k1_$dt python tools/profile_k1.py --dtype $dt --L 6 > gpurun_out/ncu_full_$dt.log 2>&1
done
echo REFRESH_DONE
