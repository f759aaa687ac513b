mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_route_gpu.py tests/test_parity_full_gpu.py tests/test_lora_gpu.py -q -x > gpurun_out/route_tests.log 2>&1; echo "rc=$?" >> gpurun_out/route_tests.log
for r in 0 16 32; do timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bgmv|sgmv|route" -c 60 --csv --log-file gpurun_out/route_ncu_$r.csv python scripts/skew_bench.py 64 1 0 $r > /dev/null 2>&1; done
