# ncu DRAM bytes of the same-data gather floor, f32 (the f64 one is in profiles/r2_floor_f64.txt)
CSEMB_PROFILE_FLOOR=1 python tools/profile_k1.py --dtype f32 --L 4 --reps 1 | tail -1
CSEMB_PROFILE_FLOOR=1 ncu --set full --clock-control none -k regex:k_diag_csr -s 1 -c 1 -f \
    -o gpurun_out/floor32 python tools/profile_k1.py --dtype f32 --L 4 --reps 1 > gpurun_out/ncu_floor32.log 2>&1
python tools/ncu_summary.py gpurun_out/floor32.ncu-rep > gpurun_out/floor_f32.txt 2>&1; cat gpurun_out/floor_f32.txt | head -14
rm -f gpurun_out/floor32.ncu-rep
