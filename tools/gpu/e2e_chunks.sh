mkdir -p gpurun_out/e2e
for c in 8 16 32; do
  timeout 600 python bench.py --e2e-chunks $c --no-cpu-baseline --no-context --c5-inst 0 > gpurun_out/e2e/c$c.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('gpurun_out/e2e/c$c.json') if l.startswith('{')][-1]); e=d['e2e']; print($c, e['value'], e['ms_per_step'], d['ms_per_step'])"
done
