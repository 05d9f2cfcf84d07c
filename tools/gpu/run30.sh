mkdir -p gpurun_out
: > gpurun_out/kbench42.log
for n in g0 gA g0 gA; do
  echo -n "$n " >> gpurun_out/kbench42.log
  KBENCH_LIB=tools/libekya_$n.so timeout 300 python tools/kbench.py grid 10 >> gpurun_out/kbench42.log 2>&1
done
timeout 600 python -m pytest tests -m gpu -q -x -k "grid or ties or config4" 2>&1 | tail -1 >> gpurun_out/kbench42.log
cat gpurun_out/kbench42.log
