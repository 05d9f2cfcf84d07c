# racecheck over the step + NEXT kernels, plus the window timeline, at small sizes
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/prof_driver.py --n-inst 512 --n-alloc 64 --n-query 256 > gpurun_out/san_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -2 gpurun_out/san_racecheck.log
KB_B=256 timeout 1500 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/win_driver.py > gpurun_out/san_race_win.log 2>&1
echo "racecheck window rc=$?"; tail -2 gpurun_out/san_race_win.log
KB_B=256 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/win_driver.py > gpurun_out/san_mem_win.log 2>&1
echo "memcheck window rc=$?"; tail -2 gpurun_out/san_mem_win.log
timeout 900 python -m pytest tests -m gpu -q -k "uniform" 2>&1 | tail -1
