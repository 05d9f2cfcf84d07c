mkdir -p gpurun_out/list
for a in "2048 256" "65536 256" "65536 64" "4096 4096" "20000 100" "300 1"; do timeout 120 python tools/list_dbg.py $a 2>&1 | tail -1; done
timeout 300 compute-sanitizer --tool memcheck python tools/list_dbg.py 2048 256 2>&1 | tail -2
timeout 300 compute-sanitizer --tool racecheck python tools/list_dbg.py 600 256 2>&1 | tail -2
timeout 300 compute-sanitizer --tool synccheck python tools/list_dbg.py 600 256 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -k "list or config4 or ties or smoke or thief" > gpurun_out/list/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/list/tests.log
tail -3 gpurun_out/list/tests.log
timeout 300 python tools/kbench.py list 10 2>&1 | tee gpurun_out/list/kbench.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list -s 2 -c 1 -o gpurun_out/list/list2 -f python tools/kbench.py list 1 > gpurun_out/list/ncu.log 2>&1
