# session 4: per-launch ncu split of one K1 step on configs 4 and 3 (fp32, final build), windows on (default) and off
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 4 3; do
 for w in auto 0; do
  if [ $w = auto ]; then unset CSEMB_HEAVY_WINDOW_MB; else export CSEMB_HEAVY_WINDOW_MB=0; fi
  python tools/profile_cfg.py --config $c --dtype f32 --L 4 > /dev/null 2>&1
  ncu --metrics $M --clock-control none -k regex:'k_step|k_heavy' -s 6 -c 3 --csv --log-file gpurun_out/s4_w_cfg${c}_$w.csv python tools/profile_cfg.py --config $c --dtype f32 --L 4 > gpurun_out/s4_w_cfg${c}_$w.log 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/s4_w_cfg${c}_$w.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
out={}
for r in rows[1:]:
    out.setdefault((r[ii], r[ki][:48]),{})[r[mi]]=float(r[vi].replace(',',''))
print('config $c fp32, column windows $w: one K1 step (ncu --clock-control none)')
tot=0
for k,v in out.items():
    tot+=v['gpu__time_duration.sum']
    print('  %-48s %7.3f ms  DRAM r/w %6.2f / %5.2f GB  L2->SM %6.2f GB  L1 hit %4.1f%%  L2 hit %4.1f%%' % (k[1], v['gpu__time_duration.sum']/1e6, v['dram__bytes_read.sum']/1e9, v['dram__bytes_write.sum']/1e9, v['l1tex__m_xbar2l1tex_read_bytes.sum']/1e9, v['l1tex__t_sector_hit_rate.pct'], v['lts__t_sector_hit_rate.pct']))
print('  total %.3f ms' % (tot/1e6))
PY
 done
done
