set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_lora_gpu.py tests/test_parity_full_gpu.py -q -x -k "bgmv or cfg1 or cfg2 or small or edge or ring or graph or compaction or linearity or delta" > gpurun_out/pytest_stream.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stream.log
for m in 1 32; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --layers-per-launch $m > gpurun_out/bench_s$m.json 2> gpurun_out/bench_s$m.err
done
timeout 300 python scripts/skew_bench.py 64 > gpurun_out/skew_s.json 2> gpurun_out/skew_s.err
