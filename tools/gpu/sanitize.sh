# compute-sanitizer memcheck / racecheck / synccheck over every kernel at small sizes
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/prof_driver.py --n-inst 512 --n-alloc 64 --n-query 256 > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_summary.log
  tail -3 gpurun_out/san_$tool.log >> gpurun_out/san_summary.log
done
cat gpurun_out/san_summary.log
