mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_lora_gpu.py tests/test_tp_gpu.py -q -x > gpurun_out/cons_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cons_tests.log
ABLATE_FLAGS=0 timeout 600 python scripts/stream_ablate.py > gpurun_out/cons_ablate.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_cons.json 2> gpurun_out/bench_cons.err
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
