# A/B of SGMV builds: cfg3 layer call (bench.py --workload cfg3) per library
for i in 1 2; do for l in "$@"; do
  PLORA_LIB=$PWD/$l timeout 300 python bench.py --workload cfg3 --steps 5 --warmup 3 --no-e2e --no-cpu > /tmp/s.json 2>/tmp/s.err
  python -c "
import json; d=json.loads(open('/tmp/s.json').readline()); print('$l', round(d['roofline']['avg_launch_us'],1), round(d['roofline']['frac'],4))" || tail -2 /tmp/s.err
done; done
