mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "place or checkpoint" > gpurun_out/gpu_tests33.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests33.log
tail -25 gpurun_out/gpu_tests33.log
