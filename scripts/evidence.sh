cd $GRAFT_REPO_ROOT
bash scripts/gpu_round.sh test,smoke,bench,launches,full,cfg3,fullsgmv
for t in memcheck racecheck synccheck; do timeout 600 compute-sanitizer --tool $t python scripts/sanitize.py > gpurun_out/sanitize_$t.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$t.log; done
timeout 600 python bench.py --workload cfg4 --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
