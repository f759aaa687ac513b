mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_gpu.py -q -x > gpurun_out/tpf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tpf_tests.log
