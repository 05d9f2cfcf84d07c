mkdir -p gpurun_out/san
for m in steepest literal; do
  KB_B=512 timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/kbench.py $m 1 > gpurun_out/san/thief_${m}_race.log 2>&1; echo "$m racecheck rc=$?"; grep SUMMARY gpurun_out/san/thief_${m}_race.log
done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/prof_driver.py --n-inst 512 --n-alloc 64 --n-query 256 > gpurun_out/san/step_racecheck2.log 2>&1; echo "step racecheck rc=$?"; grep SUMMARY gpurun_out/san/step_racecheck2.log
for m in steepest literal; do timeout 300 python tools/kbench.py $m 10; done
