# A/B of builds on the cfg5 TP numbers (bench.py --workload cfg5)
for i in 1 2; do for l in "$@"; do
  PLORA_LIB=$PWD/$l timeout 300 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-e2e --no-cpu > /tmp/c5.json 2>/tmp/c5.err
  python -c "
import json; d=json.loads(open('/tmp/c5.json').readline()); print('$l', round(d['roofline']['avg_launch_us'],1), round(d['tp_halves_at_tp1']['us_per_call'],1), round(d['tp_fused_allgather_at_tp1']['us_per_call'],1), {k:round(v['us_per_call'],1) for k,v in d['tp_rank0_halves'].items() if k!='note'})" || tail -2 /tmp/c5.err
done; done
