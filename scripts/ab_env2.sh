# A/B of an environment knob on the cfg2 decode bench: bash scripts/ab_env2.sh VAR v1 v2 ...
var=$1; shift
for i in 1 2; do for v in "$@"; do
  env $var=$v python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > /tmp/ab.json 2>/tmp/ab.err
  python -c "
import json; d=json.loads(open('/tmp/ab.json').readline())
print('$var=$v', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), round(d['per_layer_launch']['avg_launch_us'],2), round(d['per_layer_launch']['roofline_frac'],4))" || tail -3 /tmp/ab.err
done; done
