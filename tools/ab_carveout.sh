# L1/shared carveout A/B on configs 2-4 (fp32): default vs max L1 (0) vs 50
for cv in default 0 50; do
  if [ $cv = default ]; then unset CSEMB_K1_CARVEOUT; else export CSEMB_K1_CARVEOUT=$cv; fi
  timeout 300 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | sed "s/^/cv=$cv /"
  timeout 200 python tools/probe_k1.py --graphs sbm --dtype f64 2>&1 | tail -2; timeout 200 python tools/probe_k1.py --graphs sbm --dtype f32 2>&1 | tail -2 | sed "s/^/cv=$cv /"
done
