# session 4: final state -- full GPU suite, smoke, then the evidence refresh
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s4_q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4_q_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/run_round2_final.sh > gpurun_out/s4_final3.log 2>&1; tail -3 gpurun_out/s4_final3.log
