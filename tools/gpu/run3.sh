mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "profile or cluster or config3" > gpurun_out/gpu_tests29.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests29.log
for k in cluster; do timeout 120 python tools/kbench.py $k 5; done > gpurun_out/kbench29.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster2 -s 2 -c 1 -o gpurun_out/cluster2h -f python tools/kbench.py cluster 1 > gpurun_out/ncu_cluster2h.log 2>&1
tail -3 gpurun_out/gpu_tests29.log; cat gpurun_out/kbench29.log
