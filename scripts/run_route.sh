mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_route_gpu.py tests/test_parity_full_gpu.py tests/test_lora_gpu.py -q -x > gpurun_out/route_tests.log 2>&1; echo "rc=$?" >> gpurun_out/route_tests.log
for r in 0 8 16 32; do timeout 300 python scripts/skew_bench.py 64 20 0 $r >> gpurun_out/route_skew.txt 2>&1; done
timeout 300 python scripts/skew_bench.py 115 20 0 16 >> gpurun_out/route_skew.txt 2>&1
timeout 300 python scripts/skew_bench.py 115 20 0 0 >> gpurun_out/route_skew.txt 2>&1
