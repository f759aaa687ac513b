cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bgmv_warp -s 4 -c 4 -o gpurun_out/warp_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-graph > gpurun_out/ncu_warp.log 2>&1
echo "ncu rc=$?"
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/sanitize_$t.log
done
