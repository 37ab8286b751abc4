# refresh_profiles.sh, then summarise on the box (ncu -i) and keep only the
# text summaries + raw metric CSVs in gpurun_out/ (the .ncu-rep files exceed
# gpurun's 64 MiB copy-back limit)
TAG=${TAG:-r2}
TAG=$TAG bash tools/refresh_profiles.sh > gpurun_out/refresh_$TAG.log 2>&1
python tools/make_profiles.py $TAG
mkdir -p gpurun_out/prof_$TAG
cp profiles/${TAG}_* profiles/k1_traffic.json gpurun_out/prof_$TAG/ 2>/dev/null
for dt in f64 f32; do
  [ -f gpurun_out/prof_${TAG}_k1_$dt.ncu-rep ] && ncu -i gpurun_out/prof_${TAG}_k1_$dt.ncu-rep --page raw --csv > gpurun_out/prof_$TAG/raw_k1_$dt.csv
done
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out; tail -3 gpurun_out/refresh_$TAG.log
