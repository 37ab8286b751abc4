# session 4: config 4 -- lower split threshold x column windows (cold term rows windowed so their gathers stay in L2)
for w in 0 64 128 192; do
  CSEMB_HEAVY_WINDOW_MB=$w timeout 600 python tools/profile_cfg.py --config 4 --dtype f32 --L 6 --split 2048,512,256,160 2>&1 | grep "K1" | sed "s/^/window=$w MB /"
done
