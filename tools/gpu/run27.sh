mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "curve or smoke" > gpurun_out/gpu_tests45.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests45.log
timeout 600 python bench.py --steps 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench45.json 2>/dev/null
tail -2 gpurun_out/gpu_tests45.log; python -c "import json; d=json.load(open('gpurun_out/bench45.json')); print(d['context']['next2_curve_fit'])"
