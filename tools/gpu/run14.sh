mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "profile or cluster or config3 or smoke" > gpurun_out/gpu_tests20.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests20.log
(timeout 120 python tools/kbench.py radius 5) > gpurun_out/kbench20.log 2>&1
tail -3 gpurun_out/gpu_tests20.log; cat gpurun_out/kbench20.log
