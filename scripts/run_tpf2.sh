mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_gpu.py -q -x > gpurun_out/tpf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tpf_tests.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
