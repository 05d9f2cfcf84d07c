mkdir -p gpurun_out/r2c
(free -g; nproc) > gpurun_out/r2c/host.txt
python -c "import paper_2012_10557_b200.build as b; b.build()"
timeout 600 python -m pytest tests -m gpu -q -x -k "gather or pareto or prune" > gpurun_out/r2c/tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/tests.log
tail -3 gpurun_out/r2c/tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2c/bench.json; grep -i "nccl" gpurun_out/r2c/bench.err | head -5
