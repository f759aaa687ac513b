mkdir -p gpurun_out
for h in 64 115; do for r in 0 24 32 48 64 96; do timeout 300 python scripts/skew_bench.py $h 20 0 $r >> gpurun_out/route_sweep.txt 2>&1; done; done
