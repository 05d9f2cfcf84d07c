mkdir -p gpurun_out/fused
timeout 900 python -m pytest tests -m gpu -q -x -k "profile or cluster or config3" > gpurun_out/fused/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/fused/tests.log
tail -3 gpurun_out/fused/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for w in both cluster radius; do timeout 300 python tools/kbench.py $w 5; done
