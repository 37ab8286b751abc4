# session 4: fp64 staged entry batches under the sustained, power-capped bench (the probes run at full clock)
for m in 0 3 0 3; do
  echo "== CSEMB_K1_TMA=$m"; CSEMB_K1_TMA=$m timeout 400 python bench.py --skip-cpu --skip-e2e --skip-downstream --skip-configs34 --skip-builders 2>&1 | grep "\[bench\]" | head -6
done
