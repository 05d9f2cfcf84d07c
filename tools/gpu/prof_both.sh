# one ncu --set full capture (source counters) of the fused A1 kernel at the bench size
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster2 -s 2 -c 1 -o gpurun_out/both -f python tools/kbench.py both 1 > gpurun_out/ncu_both.log 2>&1
tail -3 gpurun_out/ncu_both.log
