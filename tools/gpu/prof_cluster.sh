mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster2 -s 2 -c 1 -o gpurun_out/cluster2 -f python tools/kbench.py cluster 1 > gpurun_out/ncu_cluster2.log 2>&1
tail -5 gpurun_out/ncu_cluster2.log
