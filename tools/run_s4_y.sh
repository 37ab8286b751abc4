# session 4: model check -- gathers of columns >= H bypass L1 (config 4: term ids are popularity ranks, so col < H = the H hottest term rows)
export CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_hotcol.so
for hb in 0 256 512 1024 4096 0 512; do
  CSEMB_HOT_COL_BELOW=$hb timeout 600 python tools/bench_configs.py --configs 4 --dtype f32 --reps 2 2>&1 | grep -o '"config": "[^"]*"\|"k1_ms_per_step": [0-9.]*' | paste - - | sed "s/^/hot_below=$hb /"
done
M=gpu__time_duration.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum
CSEMB_HOT_COL_BELOW=512 ncu --metrics $M --clock-control none -k regex:'k_step|k_heavy' -s 6 -c 3 --csv --log-file gpurun_out/s4_y_hot512.csv python tools/profile_cfg.py --config 4 --dtype f32 --L 4 > /dev/null 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/s4_y_hot512.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
out={}
for r in rows[1:]:
    out.setdefault((r[ii], r[ki][:48]),{})[r[mi]]=float(r[vi].replace(',',''))
for k,v in out.items():
    print('  hot_below=512 %-48s %7.3f ms  DRAM r %6.2f GB  L2->SM %6.2f GB  L1 hit %4.1f%%  L2 hit %4.1f%%' % (k[1], v['gpu__time_duration.sum']/1e6, v['dram__bytes_read.sum']/1e9, v['l1tex__m_xbar2l1tex_read_bytes.sum']/1e9, v['l1tex__t_sector_hit_rate.pct'], v['lts__t_sector_hit_rate.pct']))
PY
