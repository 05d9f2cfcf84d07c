mkdir -p gpurun_out
./tools/micro/fp2 > gpurun_out/fp2.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "profile or cluster or config3" > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests2.log
for k in cluster radius; do timeout 120 python tools/kbench.py $k 5; done > gpurun_out/kbench2.log 2>&1
cat gpurun_out/fp2.log; tail -15 gpurun_out/gpu_tests2.log; cat gpurun_out/kbench2.log
