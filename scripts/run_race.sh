mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_gpu.py -q -x > gpurun_out/tp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tp_tests.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
