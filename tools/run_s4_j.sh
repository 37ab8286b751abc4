# session 4: staged batches for fp32 4-lane groups on by default -- full GPU suite, config-1 timing, d=40 probe
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_j_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_j_pytest.log
python tools/c1time.py
CSEMB_K1_TMA=0 python tools/c1time.py | sed 's/^/TMA=0 /'
timeout 300 python tools/probe_k1.py --dtype f32 --graphs sbm,random --widths 80,40,20 --L 20 2>&1 | grep K1
python -c "import __graft_entry__ as g; g.smoke()"
