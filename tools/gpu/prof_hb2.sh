mkdir -p gpurun_out/hb
EKYA_CLUSTER_HB=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster -s 2 -c 1 -o gpurun_out/hb/hb -f python tools/kbench.py cluster 1 > gpurun_out/hb/ncu_hb.log 2>&1
tail -2 gpurun_out/hb/ncu_hb.log
