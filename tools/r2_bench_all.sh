# default bench (config 2, all legs) + configs 3/4/5 device/e2e numbers
python -c "import __graft_entry__; __graft_entry__.build()" || exit 1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/ball_c2.json 2> gpurun_out/ball_c2.err; echo "c2 rc=$?"
for c in ${CONFIGS:-4 3 5}; do
  timeout 1500 python bench.py --config $c --steps ${STEPS:-3} --warmup 3 --no-cpu > gpurun_out/ball_c$c.json 2> gpurun_out/ball_c$c.err; echo "c$c rc=$?"
done
for f in gpurun_out/ball_c*.json; do python - "$f" <<'PY'
import json,sys
d=json.load(open(sys.argv[1]))
e=d.get('e2e') or {}; p=d.get('e2e_from_posteriors') or {}
print(sys.argv[1], round(d['value']), 'ms', round(d['ms_per_step'],1), 'e2e', round(e.get('value',0)), 'post', round(p.get('value',0)), 'frac', round(d['roofline']['frac'],4), 'parity', d.get('parity'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
PY
done
