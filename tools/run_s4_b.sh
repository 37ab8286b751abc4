# session 4: K1 with the column-index / value batches staged in shared memory (CSEMB_K1_TMA=3) vs the register/shuffle default
echo "== parity with CSEMB_K1_TMA=3"
CSEMB_K1_TMA=3 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
for m in 0 3; do
  echo "== CSEMB_K1_TMA=$m"
  CSEMB_K1_TMA=$m timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm,random --widths 80,40 --L 20 2>&1 | grep K1
done
done
for m in 0 3; do
  CSEMB_K1_TMA=$m timeout 400 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/tma=$m /"
done
