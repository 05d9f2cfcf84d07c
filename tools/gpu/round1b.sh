# Round-1 evidence refresh: bench line, ncu launch list, one --set full capture per hot kernel.
mkdir -p gpurun_out/r1g
timeout 600 python bench.py > gpurun_out/r1g/bench.json 2>gpurun_out/r1g/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list_kernel|thief_kernel" --csv --log-file gpurun_out/r1g/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context > gpurun_out/r1g/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cluster2|radius_kernel|grid_kernel|list_kernel|thief_kernel|place_kernel|uniform_kernel|pareto_kernel|prune_|curve_fit_kernel|checkpoint_kernel" -c 12 -o gpurun_out/r1g/full -f python tools/prof_driver.py > gpurun_out/r1g/full.log 2>&1
tail -2 gpurun_out/r1g/full.log
python -c "import json; d=json.load(open('gpurun_out/r1g/bench.json')); print(d['value'], d['ms_per_step'], d['clocks'], d['roofline']['kernel'], d['roofline']['frac']); [print(k, round(v['ms_per_launch'],3), round(v.get('hbm_frac',0),3), round(v.get('alu_frac',0),3)) for k,v in d['rows'].items()]"
