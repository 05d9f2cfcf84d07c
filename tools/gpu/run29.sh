mkdir -p gpurun_out
: > gpurun_out/kbench41.log
for n in g0 g3 g0 g3; do for m in steepest literal; do
  echo -n "$n " >> gpurun_out/kbench41.log
  KBENCH_LIB=tools/libekya_$n.so timeout 300 python tools/kbench.py $m 10 >> gpurun_out/kbench41.log 2>&1
done; done
cat gpurun_out/kbench41.log
