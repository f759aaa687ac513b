# Diagnostics: decode step time for A/B builds of the cluster kernel's ring
# geometry (scripts/bin/libplora_j<jobbufs>_a<aslots>.so, loaded via PLORA_LIB).
set -u
for lib in scripts/bin/libplora_j*.so; do
  PLORA_LIB=$PWD/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/sweep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sweep.json')); print('$lib', round(d['roofline']['frac'],4), round(d['roofline']['avg_launch_us'],1), round(d['per_layer_launch']['roofline_frac'],4), round(d['per_layer_launch']['avg_launch_us'],2))"
done
