# fp32 rows of 320-384 bytes: 8 lanes x 3 vectors (target 3, shipped) vs 16 lanes x 2 vectors (target 2)
for v in 3 2 3 2; do
  echo "== target vpl $v"; CSEMB_TARGET_VPL=$v timeout 300 python tools/probe_k1.py --dtype f32,f64 --graphs sbm,random --widths 80,96 --L 20 2>&1 | grep K1
done
