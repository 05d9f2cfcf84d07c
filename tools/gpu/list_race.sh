mkdir -p gpurun_out/list
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/list_dbg.py 300 256 > gpurun_out/list/race.txt 2>&1
grep -E "Error|Warning|at .*eval.cu|by thread|Write|Read" gpurun_out/list/race.txt | head -60
