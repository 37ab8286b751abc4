# session 4: 5 vectors per lane on 8-lane groups (fp64 d=80: 40 vectors = 8 x 5, every lane slot used) under the sustained bench
export CSEMB_LIB_PATH=$PWD/paper_1509_08360_b200/libcsemb_cuda_wide.so
for t in 3 5 3 5; do
  echo "== target vpl $t"; CSEMB_TARGET_VPL=$t timeout 400 python bench.py --skip-cpu --skip-e2e --skip-downstream --skip-configs34 --skip-builders 2>&1 | grep "\[bench\] f"
done
