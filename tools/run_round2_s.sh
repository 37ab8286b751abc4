# compute-sanitizer over every K1 schedule path + the round-2 paths (split exchange, value-free check, gather floor)
timeout 300 python tools/sanitize_k1.py > gpurun_out/s_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/s_plain.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_k1.py > gpurun_out/s_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/s_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_k1.py > gpurun_out/s_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/s_racecheck.log
