#!/usr/bin/env bash
# End-of-session evidence on one B200: GPU tests, smoke, bench lines (cfg2, cfg3, cfg5, cfg4, reference),
# ncu launch lists + full captures (per-layer decode with split pairs, TP warp halves), sanitizers.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --workload cfg4 --steps 20 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"bgmv" -c 40 --csv --log-file $O/launches_layer.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --layers-per-launch 1 > $O/launches_layer.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bgmv_warp -s 64 -c 2 -o $O/warp_layer_full -f \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph --layers-per-launch 1 > $O/ncu_warp_layer.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bgmv_warp_tp -s 200 -c 2 -o $O/tp_full -f \
  python bench.py --workload cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_tp.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize.py > $O/sanitize_$t.log 2>&1
  echo "rc=$?" >> $O/sanitize_$t.log
done
ls -la $O
