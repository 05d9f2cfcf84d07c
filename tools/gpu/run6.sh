mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests9.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests7.log
(for n in 32 4096; do KB_N=$n timeout 120 python tools/kbench.py list 5; done; timeout 120 python tools/kbench.py grid 5) > gpurun_out/kbench9.log 2>&1
tail -3 gpurun_out/gpu_tests9.log; cat gpurun_out/kbench9.log
