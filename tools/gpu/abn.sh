# A/B/n variant builds on one kernel, interleaved twice: bash tools/gpu/abn.sh <kernel> <lib>...
mkdir -p gpurun_out
: > gpurun_out/abn.log
k=$1; shift
for rep in 1 2; do for n in "$@"; do
  echo -n "$n " >> gpurun_out/abn.log
  KBENCH_LIB=$n timeout 300 python tools/kbench.py $k 10 >> gpurun_out/abn.log 2>&1
done; done
cat gpurun_out/abn.log
