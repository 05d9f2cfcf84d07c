mkdir -p gpurun_out/r1b
timeout 900 python -m pytest tests -m gpu -x -q -k "thief or config4 or smoke" > gpurun_out/gpu_tests13.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests13.log
(for k in steepest literal; do timeout 120 python tools/kbench.py $k 5; done) > gpurun_out/kbench13.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list_kernel|thief_kernel" --csv --log-file gpurun_out/r1b/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context > gpurun_out/r1b/launches.log 2>&1
tail -2 gpurun_out/gpu_tests13.log; cat gpurun_out/kbench13.log; grep -c gpu__time gpurun_out/r1b/launches.csv
