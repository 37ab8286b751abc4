# session 4: windows for moderately heavy rows -- config 3 check and config 4 repeats
for cfg in "0 0" "64 16384" "64 65536" "0 0" "64 16384"; do
  set -- $cfg
  CSEMB_HEAVY_WINDOW_MB=$1 CSEMB_HEAVY_WINDOW_MAXLEN=$2 timeout 600 python tools/profile_cfg.py --config 3 --dtype f32 --L 6 --split 2048,256 2>&1 | grep "K1" | sed "s/^/window=$1 MB maxlen=$2 /"
  CSEMB_HEAVY_WINDOW_MB=$1 CSEMB_HEAVY_WINDOW_MAXLEN=$2 timeout 600 python tools/profile_cfg.py --config 4 --dtype f32 --L 6 --reps 2 --split 2048,256,384 2>&1 | grep "K1" | sed "s/^/window=$1 MB maxlen=$2 /"
done
