# session 4: per-kernel split of one config-4 step with / without hot-row windows (ncu, few metrics)
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum
for cfg in "0 256" "256 256"; do
  set -- $cfg
  CSEMB_HOT_ROWS=$1 CSEMB_HOT_WINDOW=$2 ncu --metrics $M --clock-control none -k regex:'k_step|k_heavy' -s 6 -c 3 --csv --log-file gpurun_out/s4_g_hot$1.csv python tools/profile_cfg.py --config 4 --dtype f32 --L 4 > gpurun_out/s4_g_hot$1.log 2>&1
  echo "hot=$1 rc=$?"
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/s4_g_hot$1.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
out={}
for r in rows[1:]:
    out.setdefault((r[ii], r[ki][:60]),{})[r[mi]]=r[vi]
for k,v in out.items(): print(k, v)
PY
done
