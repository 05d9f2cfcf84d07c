mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "profile or radius or config3 or smoke" > gpurun_out/gpu_tests39.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests39.log
(timeout 120 python tools/kbench.py radius 5) > gpurun_out/kbench39.log 2>&1
tail -2 gpurun_out/gpu_tests39.log; cat gpurun_out/kbench39.log
