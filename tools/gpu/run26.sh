mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests41.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests41.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke41.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke41.log
timeout 900 python bench.py > gpurun_out/bench41.json 2>gpurun_out/bench41.err; echo "bench rc=$?"
tail -3 gpurun_out/gpu_tests41.log; tail -2 gpurun_out/smoke41.log
python -c "import json; d=json.load(open('gpurun_out/bench41.json')); print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['clocks'], d['gpu_launches']); print(d['context'].get('next1_window'))"
tail -3 gpurun_out/bench41.err
