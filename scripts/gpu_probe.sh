# Ad-hoc GPU probe: ring trace + cfg4 bench.
mkdir -p gpurun_out
timeout 180 python scripts/trace_bgmv.py > gpurun_out/trace.txt 2>&1; echo "trace rc=$?" >> gpurun_out/trace.txt
timeout 400 python bench.py --workload cfg4 --steps 30 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "rc=$?" >> gpurun_out/bench_cfg4.err
