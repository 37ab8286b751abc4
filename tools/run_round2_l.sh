# ncu --set full: the gather floor vs K1 (shipped) vs K1 without epilogue streams (ab5), fp64 config 2
mkdir -p gpurun_out/l
CSEMB_PROFILE_FLOOR=1 python tools/profile_k1.py --dtype f64 --L 4 --reps 1
CSEMB_PROFILE_FLOOR=1 ncu --set full --clock-control none --import-source on -k regex:k_diag_csr -s 1 -c 1 -f -o gpurun_out/l/floor python tools/profile_k1.py --dtype f64 --L 4 --reps 1 > gpurun_out/l/ncu_floor.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -f -o gpurun_out/l/k1 python tools/profile_k1.py --dtype f64 --L 6 > gpurun_out/l/ncu_k1.log 2>&1
CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_ab5.so ncu --set full --clock-control none --import-source on -k regex:k_step -s 3 -c 1 -f -o gpurun_out/l/k1ab5 python tools/profile_k1.py --dtype f64 --L 6 > gpurun_out/l/ncu_ab5.log 2>&1
for r in floor k1 k1ab5; do
  ncu -i gpurun_out/l/$r.ncu-rep --page raw --csv > gpurun_out/l/raw_$r.csv
  ncu -i gpurun_out/l/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/l/src_$r.csv 2>/dev/null
  ncu -i gpurun_out/l/$r.ncu-rep --page details > gpurun_out/l/details_$r.txt
done
python tools/ncu_summary.py gpurun_out/l/floor.ncu-rep gpurun_out/l/k1.ncu-rep gpurun_out/l/k1ab5.ncu-rep
rm -f gpurun_out/l/*.ncu-rep
