# Round-2 re-entry evidence: full GPU tests + smoke, bench line, launch list, CLUSTER A/B, ncu full of the hot kernels.
mkdir -p gpurun_out/r2e
nproc > gpurun_out/r2e/host.txt; free -g >> gpurun_out/r2e/host.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2e/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2e/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2e/smoke.log
tail -3 gpurun_out/r2e/tests.log; tail -2 gpurun_out/r2e/smoke.log
timeout 900 python bench.py > gpurun_out/r2e/bench.json 2>gpurun_out/r2e/bench.err; echo "bench rc=$?"
for v in 0 1; do if [ $v = 1 ]; then export EKYA_CLUSTER_HB=1; fi; echo "HB=$v"; timeout 300 python tools/kbench.py cluster 5; done > gpurun_out/r2e/kbench_cluster.txt 2>&1
unset EKYA_CLUSTER_HB
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list_kernel|thief_kernel" --csv --log-file gpurun_out/r2e/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context --c5-inst 0 > gpurun_out/r2e/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cluster2|radius_kernel|grid_kernel|list_kernel|thief_kernel" -c 6 -o gpurun_out/r2e/full -f python tools/prof_driver.py > gpurun_out/r2e/full.log 2>&1
tail -2 gpurun_out/r2e/full.log
cat gpurun_out/r2e/kbench_cluster.txt
