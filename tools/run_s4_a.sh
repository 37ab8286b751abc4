# session 4: K1 variants on the skewed full-scale configs (fp32): gather prefetch, depth 4, 3 CTAs/SM
for v in "" pf d4 mb3; do
  if [ -n "$v" ]; then export CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_$v.so; else unset CSEMB_LIB_PATH; fi
  timeout 400 python tools/bench_configs.py --configs 4,3 --dtype f32 --reps 2 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        j = json.loads(l); print('variant=${v:-base}', j['config'], j['dtype'], 'K1', j['k1_ms_per_step'], 'ms/step embed', j['embed_ms'])
    else: print(l.rstrip()[:200])
"
done
