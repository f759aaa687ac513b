mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sgmv_gpu.py tests/test_parity_full_gpu.py -q -x > gpurun_out/sgmv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sgmv_tests.log
timeout 500 python scripts/sgmv_ablate.py > gpurun_out/sgmv_ablate.txt 2>&1
timeout 600 python bench.py --workload cfg3 --steps 10 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
