mkdir -p gpurun_out
for n in 8 9 10 8 9 10; do for m in steepest literal; do
  echo -n "t$n " >> gpurun_out/kbench40.log
  KBENCH_LIB=tools/libekya_t$n.so timeout 300 python tools/kbench.py $m 10 >> gpurun_out/kbench40.log 2>&1
done; done
cat gpurun_out/kbench40.log
