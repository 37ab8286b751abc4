# session 4: fp32 gather depth 4 on top of index staging (spill-free now)
for v in "" d4 "" d4; do
  if [ -n "$v" ]; then export CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_$v.so; else unset CSEMB_LIB_PATH; fi
  echo "== variant ${v:-default}"
  timeout 300 python tools/probe_k1.py --dtype f32 --graphs sbm,random --widths 80,40,20,10 --L 20 2>&1 | grep K1
  timeout 400 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - -
done
