timeout 400 python -m pytest tests/test_tp_gpu.py -q > gpurun_out/pt_tp.log 2>&1; tail -1 gpurun_out/pt_tp.log
timeout 400 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5_warp.json 2> gpurun_out/bench_cfg5_warp.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bgmv_warp_tp" -c 200 --csv --log-file gpurun_out/tp_launches.csv python bench.py --workload cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/tp_launches.log 2>&1
