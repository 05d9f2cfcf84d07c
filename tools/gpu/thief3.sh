mkdir -p gpurun_out/thief
timeout 900 python -m pytest tests -m gpu -q -x -k "thief or window or config4 or config5 or gather or ties or place or profile_output" > gpurun_out/thief/tests3.log 2>&1; echo "tests rc=$?" >> gpurun_out/thief/tests3.log
tail -3 gpurun_out/thief/tests3.log
for m in steepest literal; do timeout 300 python tools/kbench.py $m 10; done
for m in steepest literal; do KB_C5=1 KB_B=16384 timeout 300 python tools/kbench.py $m 5; done
