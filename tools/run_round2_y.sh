# config 5 on an R x C grid, one rank's share on one B200: R row blocks (--gpus R), d/C columns per rank
for rc in "8 64" "4 32" "2 16"; do
  set -- $rc
  timeout 900 python tools/bench_config5_rank.py --gpus $1 --d $2 --steps 6 --out gpurun_out/y_grid_$1x$((64/$2)).json > gpurun_out/y_grid_$1.log 2>&1
  echo "R=$1 d_local=$2 rc=$?"; tail -c 700 gpurun_out/y_grid_$1.log; echo
done
