mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "window" > gpurun_out/gpu_tests40.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests40.log
tail -30 gpurun_out/gpu_tests40.log
