# A/B of decode builds on one box: bash scripts/ab_decode.sh <lib.so | repo-dir> ...
# (a dir holds a full checkout with its libplora.so built in place; a .so
# is loaded through PLORA_LIB with this checkout's Python)
for t in "$@"; do
  if [ -d "$t" ]; then
    (cd $t && python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > /tmp/ab.json 2>/tmp/ab.err)
  else
    PLORA_LIB=$PWD/$t python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > /tmp/ab.json 2>/tmp/ab.err
  fi
  python -c "
import json; d=json.loads(open('/tmp/ab.json').readline())
print('$t', round(d['ms_per_step'],4), round(d['roofline']['frac'],4), round(d['per_layer_launch']['avg_launch_us'],2), round(d['per_layer_launch']['roofline_frac'],4))" || tail -3 /tmp/ab.err
done
