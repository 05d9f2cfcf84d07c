mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "curve" > gpurun_out/gpu_tests36.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests36.log
tail -25 gpurun_out/gpu_tests36.log
