mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench4.log 2>gpurun_out/bench4.err; echo "bench rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list_kernel -s 2 -c 1 -o gpurun_out/list -f python tools/kbench.py list 1 > gpurun_out/ncu_list.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 2 -c 1 -o gpurun_out/grid -f python tools/kbench.py grid 1 > gpurun_out/ncu_grid.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/steepest -f python tools/kbench.py steepest 1 > gpurun_out/ncu_steep.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/literal -f python tools/kbench.py literal 1 > gpurun_out/ncu_lit.log 2>&1
cat gpurun_out/bench4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks']); [print(k, round(v['ms_per_launch'],3), round(v.get('hbm_frac',0),3)) for k,v in d['rows'].items()]"
