#!/usr/bin/env bash
# Round-end evidence on one GPU box (run through gpurun): tests, smoke, the
# bench lines of every workload, ncu launch list + full captures, sanitizers.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
bash scripts/gpu_round.sh test,smoke,bench,launches,full,cfg3,fullsgmv,fused
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python scripts/sanitize.py > gpurun_out/sanitize_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$t.log
done
timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
