mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "grid or config4 or smoke or ties" > gpurun_out/gpu_tests38.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests11.log
(timeout 120 python tools/kbench.py grid 5) > gpurun_out/kbench38.log 2>&1
tail -2 gpurun_out/gpu_tests38.log; cat gpurun_out/kbench38.log
