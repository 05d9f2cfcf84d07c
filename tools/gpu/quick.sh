# quick check: a -k subset of the GPU tests and the bench context rows
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "$1" > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/quick_bench.json 2>/dev/null
tail -2 gpurun_out/quick_tests.log; python -c "import json,sys; d=json.load(open('gpurun_out/quick_bench.json')); [print(k, d['context'][k]) for k in sys.argv[1:]]" $2
