mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests28.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests28.log
tail -15 gpurun_out/gpu_tests28.log
