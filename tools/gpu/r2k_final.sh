# round-2 final: full GPU tests + smoke, launch list, ncu --set full of the hot kernels
mkdir -p gpurun_out/r2k3
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2k3/gpu_full.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2k3/gpu_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2k3/smoke.log
tail -2 gpurun_out/r2k3/gpu_full.log; tail -2 gpurun_out/r2k3/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list|thief_kernel" --csv --log-file gpurun_out/r2k3/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context --c5-inst 0 > gpurun_out/r2k3/launches.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"cluster2|grid_kernel|list|thief_kernel" -c 5 -o gpurun_out/r2k3/full -f python tools/prof_driver.py --no-next > gpurun_out/r2k3/full.log 2>&1; echo "full rc=$?"
