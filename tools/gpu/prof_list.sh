mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list_kernel -s 2 -c 1 -o gpurun_out/list6 -f python tools/kbench.py list 1 > gpurun_out/ncu_list6.log 2>&1
KB_N=32 timeout 300 ncu --set full --clock-control none --import-source on -k regex:list_kernel -s 2 -c 1 -o gpurun_out/list6_n32 -f python tools/kbench.py list 1 > gpurun_out/ncu_list6n.log 2>&1
tail -2 gpurun_out/ncu_list6.log
