# racecheck + memcheck over the generic kernel instantiations exercised by parity tests
mkdir -p gpurun_out
K="odd or wide or bigU or v1 or big-h or h513 or h256 or c32 or prune_random"
for tool in racecheck memcheck; do
  timeout 2400 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/san3_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "passed|failed|SUMMARY" gpurun_out/san3_$tool.log | tail -3
done
