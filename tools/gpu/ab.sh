# A/B two variant builds on one kernel: bash tools/gpu/ab.sh <kernel> <libA> <libB>
mkdir -p gpurun_out
: > gpurun_out/ab.log
for n in $2 $3 $2 $3; do
  echo -n "$n " >> gpurun_out/ab.log
  KBENCH_LIB=$n timeout 300 python tools/kbench.py $1 10 >> gpurun_out/ab.log 2>&1
done
cat gpurun_out/ab.log
