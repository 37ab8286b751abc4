# session 4: variant parity tests; entry batches via LDG.cs -> registers -> STS (CSEMB_K1_TMA=4) vs cp.async (3) vs shuffles (0)
timeout 1500 python -m pytest tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -5
CSEMB_K1_TMA=4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for rep in 1 2; do
for m in 0 3 4; do
  echo "== CSEMB_K1_TMA=$m"
  CSEMB_K1_TMA=$m timeout 300 python tools/probe_k1.py --dtype f64,f32 --graphs sbm,random --widths 80 --L 20 2>&1 | grep K1
done
done
for m in 3 4; do
  CSEMB_K1_TMA=$m timeout 400 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/tma=$m /"
done
