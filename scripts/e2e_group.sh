for i in 1 2; do for g in ${EG:-1 2 4 8}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --e2e-group $g > /tmp/e.json 2>/tmp/e.err
  python -c "
import json; d=json.loads(open('/tmp/e.json').readline()); print('group $g', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],3))" || tail -2 /tmp/e.err
done; done
