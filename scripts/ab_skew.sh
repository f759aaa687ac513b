# A/B of decode builds on the skewed and uniform 512-token batches (scripts/skew_bench.py) and the cfg2 bench
for i in 1 2; do for l in "$@"; do
  PLORA_LIB=$PWD/$l timeout 200 python scripts/skew_bench.py 115 20 0 160 > /tmp/sk.json 2>/tmp/sk.err
  python -c "
import json; d=json.loads(open('/tmp/sk.json').readline()); print('$l skew', round(d['skewed']['us_per_layer_launch'],1), 'uniform', round(d['uniform']['us_per_layer_launch'],1))" || tail -2 /tmp/sk.err
done; done
bash scripts/ab_decode.sh "$@"
