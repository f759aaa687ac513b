# quick decode bench + launch split (run on the GPU box)
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/b.json 2>gpurun_out/b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bgmv" -c 400 --csv --log-file gpurun_out/l.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python - <<'PY'
import json, csv, collections
d=json.loads(open('gpurun_out/b.json').readline())
print("step_ms", round(d['ms_per_step'],4), "frac", round(d['roofline']['frac'],4), "per_layer_us", round(d['per_layer_launch']['avg_launch_us'],2), "pl_frac", round(d['per_layer_launch']['roofline_frac'],4), "e2e", (d['e2e'] or {}).get('value'))
rows=[r for r in csv.reader(open('gpurun_out/l.csv')) if len(r)>5]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); gi=h.index('Grid Size')
dd=collections.defaultdict(list)
for r in rows[1:]:
    try: dd[(r[ki][25:60], r[gi])].append(float(r[vi].replace(',','')))
    except: pass
for k,v in dd.items(): print(k, len(v), round(sum(v)/len(v)/1000,2), 'us')
PY
