mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench23.json 2>gpurun_out/bench23.err; echo "bench rc=$?"
tail -2 gpurun_out/smoke.log
python -c "import json; d=json.load(open('gpurun_out/bench23.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['clocks']); print({k: v for k, v in d['context'].items() if k.startswith('next')}); print(d['cpu_baseline'])"
tail -3 gpurun_out/bench23.err
