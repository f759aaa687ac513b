#!/usr/bin/env bash
# One GPU session: tests, smoke, bench, ncu launch list + one full capture.
# Usage (from this container):  gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh [stages]'
# stages: any of test,smoke,bench,launches,full,cfg3,fullsgmv,fused (default: the first five)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
STAGES="${1:-test,smoke,bench,launches,full}"
has() { [[ ",$STAGES," == *",$1,"* ]]; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/host_cores.txt; lscpu | grep -i "model name" >> gpurun_out/host_cores.txt
if has test; then
  timeout 600 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke rc=$?" >> gpurun_out/smoke.log
fi
if has bench; then
  timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
if has launches; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bgmv|sgmv|page_" -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/launches.log 2>&1
  echo "launches rc=$?" >> gpurun_out/launches.log
fi
if has full; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bgmv_cluster -s 100 -c 2 \
    -o gpurun_out/bgmv_full -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_full.log 2>&1
  echo "full rc=$?" >> gpurun_out/ncu_full.log
fi
if has cfg3; then
  timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
  echo "cfg3 rc=$?" >> gpurun_out/bench_cfg3.err
fi
if has fullsgmv; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_ -s 70 -c 3 \
    -o gpurun_out/sgmv_full -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-e2e --no-cpu \
    > gpurun_out/ncu_sgmv.log 2>&1
  echo "fullsgmv rc=$?" >> gpurun_out/ncu_sgmv.log
fi
ls -la gpurun_out
if has fused; then
  timeout 600 python bench.py --workload cfg3f --steps 5 --warmup 3 > gpurun_out/bench_cfg3f.json 2> gpurun_out/bench_cfg3f.err
  echo "cfg3f rc=$?" >> gpurun_out/bench_cfg3f.err
  timeout 300 python scripts/fused_bench.py > gpurun_out/fused_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgmv_fused -s 20 -c 1 \
    -o gpurun_out/fused_full -f python scripts/fused_bench.py > gpurun_out/ncu_fused.log 2>&1
  echo "fused rc=$?" >> gpurun_out/ncu_fused.log
fi
