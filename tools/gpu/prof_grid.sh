mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 2 -c 1 -o gpurun_out/grid4 -f python tools/kbench.py grid 1 > /dev/null 2>&1
ls gpurun_out/grid4.ncu-rep
