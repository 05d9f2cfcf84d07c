# A/B/C three variant builds on one kernel: bash tools/gpu/ab3.sh <kernel> <libA> <libB> <libC>
mkdir -p gpurun_out
: > gpurun_out/ab3.log
for n in $2 $3 $4 $2 $3 $4; do
  echo -n "$n " >> gpurun_out/ab3.log
  KBENCH_LIB=$n timeout 300 python tools/kbench.py $1 10 >> gpurun_out/ab3.log 2>&1
done
cat gpurun_out/ab3.log
