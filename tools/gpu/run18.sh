mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "grid or list or config4 or smoke or feeds" > gpurun_out/gpu_tests27.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests27.log
(for k in grid list; do timeout 120 python tools/kbench.py $k 5; done) > gpurun_out/kbench27.log 2>&1
tail -2 gpurun_out/gpu_tests27.log; cat gpurun_out/kbench27.log
