# thief A/B: parity of every thief-driven test, then kernel timings (config 4 both modes, config-5 shape)
mkdir -p gpurun_out/thief
timeout 900 python -m pytest tests -m gpu -q -x -k "thief or window or config4 or config5 or gather or ties or place or profile_output" > gpurun_out/thief/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/thief/tests.log
tail -3 gpurun_out/thief/tests.log
for m in steepest literal; do timeout 300 python tools/kbench.py $m 10; done 2>&1 | tee gpurun_out/thief/kbench.txt
for m in steepest literal; do KB_C5=1 KB_B=16384 timeout 300 python tools/kbench.py $m 5; done 2>&1 | tee -a gpurun_out/thief/kbench.txt
if [ -f paper_2012_10557_b200/libekya_old.so ]; then
  for m in steepest literal; do KBENCH_LIB=paper_2012_10557_b200/libekya_old.so timeout 300 python tools/kbench.py $m 10; done 2>&1 | tee -a gpurun_out/thief/kbench.txt
  for m in steepest literal; do KB_C5=1 KB_B=16384 KBENCH_LIB=paper_2012_10557_b200/libekya_old.so timeout 300 python tools/kbench.py $m 5; done 2>&1 | tee -a gpurun_out/thief/kbench.txt
fi
