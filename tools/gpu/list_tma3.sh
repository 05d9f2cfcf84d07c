mkdir -p gpurun_out/list
for a in "2048 256" "20000 100" "300 1" "3000 77" "65536 4096"; do timeout 120 python tools/list_dbg.py $a 2>&1 | tail -1; done
timeout 600 python -m pytest tests -m gpu -q -x -k "list or config4 or ties" 2>&1 | tail -2
timeout 300 python tools/kbench.py list 10
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list -s 2 -c 1 -o gpurun_out/list/list2c -f python tools/kbench.py list 1 > gpurun_out/list/ncu.log 2>&1
