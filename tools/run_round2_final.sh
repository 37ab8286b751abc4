# Round-2 final evidence: bench line (ours + reference arm), ncu launch list, ncu --set full of K1 (f64/f32)
# and of the same-data gather floor; summaries into gpurun_out/prof_r2 (copied to profiles/ afterwards)
TAG=r2 bash tools/refresh_and_summarise.sh
CSEMB_PROFILE_FLOOR=1 ncu --set full --clock-control none --import-source on -k regex:k_diag_csr -s 1 -c 1 -f \
    -o gpurun_out/floor_r2 python tools/profile_k1.py --dtype f64 --L 4 --reps 1 > gpurun_out/ncu_floor_r2.log 2>&1
python tools/ncu_summary.py gpurun_out/floor_r2.ncu-rep > gpurun_out/prof_r2/floor_f64.txt 2>&1
rm -f gpurun_out/floor_r2.ncu-rep
cp gpurun_out/bench_r2.json gpurun_out/bench_ref_r2.json gpurun_out/prof_r2/ 2>/dev/null
tail -c 400 gpurun_out/bench_r2.json; echo; tail -c 300 gpurun_out/bench_ref_r2.json; echo
