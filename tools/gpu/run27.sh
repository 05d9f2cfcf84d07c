mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "prune or pareto or abi" > gpurun_out/gpu_tests49.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests49.log
timeout 600 python bench.py --steps 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench49.json 2>/dev/null
tail -2 gpurun_out/gpu_tests49.log; python -c "import json; d=json.load(open('gpurun_out/bench49.json')); print(d['context']['next3_prune'])"
