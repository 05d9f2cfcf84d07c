mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench15.json 2>gpurun_out/bench15.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench15.json')); print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['frac']); [print(k, round(v['ms_per_launch'],3)) for k,v in d['rows'].items()]"
tail -3 gpurun_out/bench15.err
