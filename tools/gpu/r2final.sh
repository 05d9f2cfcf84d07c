# round-2 re-entry check: full GPU tests + smoke + bench line at HEAD
mkdir -p gpurun_out/r2f
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2f/gpu_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2f/gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2f/smoke.log
timeout 900 python bench.py > gpurun_out/r2f/bench.json 2>gpurun_out/r2f/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2f/gpu_full.log; tail -2 gpurun_out/r2f/smoke.log
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2f/bench.json') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'], d['e2e']['value'])
[print(k, round(v['ms_per_launch'],3), v.get('hbm_frac'), v.get('alu_frac'), v.get('issue_frac')) for k,v in d['rows'].items()]
"
