mkdir -p gpurun_out
ABLATE_FLAGS=0,1 timeout 600 python scripts/stream_ablate.py > gpurun_out/pf_ablate.txt 2>&1
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.err
timeout 900 python -m pytest tests/test_tp_gpu.py tests/test_lora_gpu.py tests/test_parity_full_gpu.py -q -x > gpurun_out/pf_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pf_tests.log
