# round 2: compute-sanitizer memcheck / racecheck / synccheck over the step's kernels (fused A1,
# list2, both thieves, GRID) + NEXT rows at small sizes, the wide (V = 100) thief, and the
# generic instantiations through the parity tests
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/prof_driver.py --n-inst 512 --n-alloc 64 --n-query 256 > gpurun_out/san/step_$tool.log 2>&1
  echo "step $tool rc=$?" | tee -a gpurun_out/san/summary.log; grep -E "SUMMARY|hazard" gpurun_out/san/step_$tool.log | tail -2 | tee -a gpurun_out/san/summary.log
done
for tool in memcheck racecheck; do
  KB_C5=1 KB_B=64 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/kbench.py steepest 1 > gpurun_out/san/c5s_$tool.log 2>&1
  echo "c5 steepest $tool rc=$?" | tee -a gpurun_out/san/summary.log; grep -E "SUMMARY" gpurun_out/san/c5s_$tool.log | tail -1 | tee -a gpurun_out/san/summary.log
  KB_C5=1 KB_B=64 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/kbench.py literal 1 > gpurun_out/san/c5l_$tool.log 2>&1
  echo "c5 literal $tool rc=$?" | tee -a gpurun_out/san/summary.log; grep -E "SUMMARY" gpurun_out/san/c5l_$tool.log | tail -1 | tee -a gpurun_out/san/summary.log
done
K="odd or wide or bigU or v1 or big-h or h513 or h256 or c32 or prune_random or both"
for tool in racecheck memcheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/san/tests_$tool.log 2>&1
  echo "tests $tool rc=$?" | tee -a gpurun_out/san/summary.log; grep -E "passed|failed|SUMMARY" gpurun_out/san/tests_$tool.log | tail -2 | tee -a gpurun_out/san/summary.log
done
grep -E "hazard detected|Write Thread|Read Thread" gpurun_out/san/step_racecheck.log | sed 's/(.*)//' | sort | uniq -c | sort -rn | head -20 > gpurun_out/san/race_sites.txt
