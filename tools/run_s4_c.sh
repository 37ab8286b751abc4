# session 4: index staging default for fp32 -- full GPU suite, then hint / two-entries-per-lane variants
timeout 2000 python -m pytest tests -m gpu -x -q > gpurun_out/s4_c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_c_pytest.log
for v in "" hint eb2; do
  if [ -n "$v" ]; then export CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_$v.so; else unset CSEMB_LIB_PATH; fi
  echo "== variant ${v:-default}"
  timeout 300 python tools/probe_k1.py --dtype f32 --graphs sbm,random --widths 80,96 --L 20 2>&1 | grep K1
  timeout 400 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - -
done
