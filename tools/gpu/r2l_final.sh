# round-2 final: full GPU tests + smoke, launch list, ncu --set full of the hot kernels
mkdir -p gpurun_out/r2l
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l/gpu_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2l/gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2l/smoke.log
tail -2 gpurun_out/r2l/gpu_full.log; tail -2 gpurun_out/r2l/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list|thief_kernel" --csv --log-file gpurun_out/r2l/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context --c5-inst 0 > gpurun_out/r2l/launches.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"cluster2|grid_kernel|list|thief_kernel" -c 5 -o gpurun_out/r2l/full -f python tools/prof_driver.py --no-next > gpurun_out/r2l/full.log 2>&1; echo "full rc=$?"
