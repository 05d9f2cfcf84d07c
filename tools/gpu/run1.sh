mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc=$?"
for k in cluster list grid radius steepest literal; do timeout 120 python tools/kbench.py $k 5; done > gpurun_out/kbench.log 2>&1
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench.log; cat gpurun_out/kbench.log
