# session 4 final evidence: refresh (bench, reference arm, launch list, K1 ncu captures, floor), config 3/4 ncu split, first-call cost
bash tools/run_round2_final.sh > gpurun_out/s4_final2.log 2>&1; tail -3 gpurun_out/s4_final2.log
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 4 3; do
  python tools/profile_cfg.py --config $c --dtype f32 --L 4 > /dev/null 2>&1
  ncu --metrics $M --clock-control none -k regex:'k_step|k_heavy' -s 6 -c 3 --csv --log-file gpurun_out/s4_cfg${c}_split.csv python tools/profile_cfg.py --config $c --dtype f32 --L 4 > gpurun_out/s4_cfg${c}_split.log 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/s4_cfg${c}_split.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
out={}
for r in rows[1:]:
    out.setdefault((r[ii], r[ki][:60]),{})[r[mi]]=r[vi]
print('config $c fp32, one K1 step (ncu):')
for k,v in out.items(): print(' ', k[1], {a.split('__')[-1]: b for a,b in v.items()})
PY
done
python - <<'PY'
import sys, time, math
sys.path.insert(0, '.')
import torch, paper_1509_08360_b200 as pb
from paper_1509_08360_b200 import _lib, device_build as db
S = db.dilate(db.bag_of_words(2_000_000, 500_000, seed=4))
dm = S.to_device_matrix("float32"); dm.scale(1.0 / 130.35983614177252)
coeffs = pb.legendre_coefficients(pb.indicator_above(0.3), 4).coeffs
plan = dm.plan(96)
for i in range(3):
    dm.ctx.sync(); t = time.perf_counter(); plan.run(coeffs, 1, omega_kind=_lib.OMEGA_PHILOX, seed=7); dm.ctx.sync()
    print(f"config 4 plan.run #{i} (L=4): {1e3*(time.perf_counter()-t):.1f} ms wall")
PY
