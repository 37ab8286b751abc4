# gather floor (csemb_diag_gather_csr) vs K1, and the reference suite with the warm-up
timeout 900 python tools/probe_floor.py --dtype f64,f32 --graphs sbm,random,band --widths 80,40,10 > gpurun_out/i_floor.log 2>&1; echo "floor rc=$?"
cat gpurun_out/i_floor.log | grep K1
timeout 600 python -m pytest tests/test_reference_suite.py -m gpu -q > gpurun_out/i_refsuite.log 2>&1; echo "refsuite rc=$?"; tail -3 gpurun_out/i_refsuite.log
