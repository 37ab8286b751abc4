# session 4: config 4 -- windows only for rows up to MAXLEN entries, lower split thresholds
for cfg in "0 0" "64 4096" "64 16384" "64 65536" "96 16384" "48 16384" "32 16384"; do
  set -- $cfg
  CSEMB_HEAVY_WINDOW_MB=$1 CSEMB_HEAVY_WINDOW_MAXLEN=$2 timeout 600 python tools/profile_cfg.py --config 4 --dtype f32 --L 6 --split 2048,256,160,128 2>&1 | grep "K1" | sed "s/^/window=$1 MB maxlen=$2 /"
done
