# one ncu --set full capture (source counters) each of LIST, GRID and the STEEPEST thief at the bench size
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list -s 2 -c 1 -o gpurun_out/list -f python tools/kbench.py list 1 > gpurun_out/ncu_list.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 2 -c 1 -o gpurun_out/grid -f python tools/kbench.py grid 1 > gpurun_out/ncu_grid.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/steep -f python tools/kbench.py steepest 1 > gpurun_out/ncu_steep.log 2>&1
ls -la gpurun_out/*.ncu-rep
