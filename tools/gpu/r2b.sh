mkdir -p gpurun_out/r2b
python -c "import paper_2012_10557_b200.build as b; b.build()"
timeout 1700 python -m pytest tests -m gpu -q -x -k "bench_launch or config5_sample or config4_full or prune" --durations=10 > gpurun_out/r2b/tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/tests.log
tail -15 gpurun_out/r2b/tests.log
