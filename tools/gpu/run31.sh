mkdir -p gpurun_out
: > gpurun_out/kbench43.log
for n in l0 lA l0 lA; do
  echo -n "$n " >> gpurun_out/kbench43.log
  KBENCH_LIB=tools/libekya_$n.so timeout 300 python tools/kbench.py list 10 >> gpurun_out/kbench43.log 2>&1
done
cat gpurun_out/kbench43.log
