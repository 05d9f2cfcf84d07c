# A1 profile parity + timing of the fused launch (and CLUSTER / RADIUS alone) at the bench size
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "profile or cluster or config3 or lloyd" > gpurun_out/ab_prof_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_prof_tests.log
tail -3 gpurun_out/ab_prof_tests.log
for w in both cluster; do timeout 300 python tools/kbench.py $w 10; done
