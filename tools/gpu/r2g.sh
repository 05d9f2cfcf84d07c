# Round-2 evidence: full GPU tests + smoke, bench line, launch list, ncu --set full of the hot kernels
mkdir -p gpurun_out/r2g
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2g/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2g/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2g/smoke.log
tail -3 gpurun_out/r2g/tests.log; tail -2 gpurun_out/r2g/smoke.log
timeout 900 python bench.py > gpurun_out/r2g/bench.json 2>gpurun_out/r2g/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list|thief_kernel" --csv --log-file gpurun_out/r2g/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context --c5-inst 0 > gpurun_out/r2g/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cluster2|radius_kernel|grid_kernel|list|thief_kernel" -c 6 -o gpurun_out/r2g/full -f python tools/prof_driver.py > gpurun_out/r2g/full.log 2>&1
tail -2 gpurun_out/r2g/full.log
