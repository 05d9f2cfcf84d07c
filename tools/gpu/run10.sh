mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "thief or config4 or smoke or feeds or ties" > gpurun_out/gpu_tests32.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests15.log
(for k in steepest literal; do timeout 120 python tools/kbench.py $k 5; done) > gpurun_out/kbench32.log 2>&1
tail -2 gpurun_out/gpu_tests32.log; cat gpurun_out/kbench32.log
