mkdir -p gpurun_out/r2d
python -c "import paper_2012_10557_b200.build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -q -x -k "profile or cluster or gather or pareto" > gpurun_out/r2d/tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/tests.log
tail -3 gpurun_out/r2d/tests.log
for v in 0 1; do if [ $v = 1 ]; then export EKYA_CLUSTER_NOHB=1; fi; python tools/kbench.py cluster 5; done 2>&1 | tee gpurun_out/r2d/kbench.txt
