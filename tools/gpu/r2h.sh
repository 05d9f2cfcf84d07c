# bench line + launch list + ncu full of the hot kernels (fused A1)
mkdir -p gpurun_out/r2h
timeout 900 python bench.py > gpurun_out/r2h/bench.json 2>gpurun_out/r2h/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cluster|radius_kernel|grid_kernel|list|thief_kernel" --csv --log-file gpurun_out/r2h/launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-context --c5-inst 0 > gpurun_out/r2h/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"cluster2|grid_kernel|list|thief_kernel" -c 5 -o gpurun_out/r2h/full -f python tools/prof_driver.py --no-next > gpurun_out/r2h/full.log 2>&1
tail -1 gpurun_out/r2h/full.log
python -c "
import json; d=json.loads([l for l in open('gpurun_out/r2h/bench.json') if l.startswith('{')][-1])
print(d['value'], d['ms_per_step'], d['roofline']['kernel'], round(d['roofline']['frac'],3), d['clocks'], d['e2e']['value'])
[print(k, round(v['ms_per_launch'],3), v.get('hbm_frac'), v.get('alu_frac'), v.get('issue_frac')) for k,v in d['rows'].items()]
"
