# session 4: 8 lanes x 5 vectors for rows of 33..40 vectors (default) vs 16 x 3 (CSEMB_WIDE_SHAPE=0): sustained bench, probes, full suite
for w in 1 0 1 0; do
  echo "== CSEMB_WIDE_SHAPE=$w"; CSEMB_WIDE_SHAPE=$w timeout 400 python bench.py --skip-cpu --skip-e2e --skip-downstream --skip-configs34 --skip-builders 2>&1 | grep "\[bench\] f"
done
for w in 1 0; do
  echo "== probe CSEMB_WIDE_SHAPE=$w"
  CSEMB_WIDE_SHAPE=$w timeout 300 python tools/probe_k1.py --dtype f64 --graphs sbm,random --widths 80,72,66 --L 20 2>&1 | grep K1
  CSEMB_WIDE_SHAPE=$w timeout 300 python tools/probe_k1.py --dtype f32 --graphs sbm,random --widths 160,144 --L 20 2>&1 | grep K1
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_bb_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_bb_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
