mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list_kernel -s 2 -c 1 -o gpurun_out/list4 -f python tools/kbench.py list 1 > gpurun_out/ncu_list4.log 2>&1
KB_N=32 timeout 300 ncu --set full --clock-control none --import-source on -k regex:list_kernel -s 2 -c 1 -o gpurun_out/list4_n32 -f python tools/kbench.py list 1 > gpurun_out/ncu_list4n.log 2>&1
tail -2 gpurun_out/ncu_list4.log
