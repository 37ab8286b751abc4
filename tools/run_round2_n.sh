# value-free normalized adjacency: GPU suite, A/B on config-2-sized graphs (widths 80/40/10), bench line
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/n_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/n_pytest.log
for rep in 1 2; do
for vf in 0 1; do
  echo "== CSEMB_VALUE_FREE=$vf"
  CSEMB_VALUE_FREE=$vf timeout 300 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random --widths 80,40,10 2>&1 | grep K1 | sed 's/| gather floor.*K1/| K1/'
done
done
timeout 900 python bench.py --skip-cpu > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo "bench rc=$?"
