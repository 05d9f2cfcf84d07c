mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "list or config4 or smoke or limits or ties" > gpurun_out/gpu_tests37.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests14.log
(for n in 32 4096; do KB_N=$n timeout 120 python tools/kbench.py list 5; done) > gpurun_out/kbench37.log 2>&1
tail -2 gpurun_out/gpu_tests37.log; cat gpurun_out/kbench37.log
