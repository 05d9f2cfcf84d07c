mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "profile or cluster or config3 or lloyd or persistent" > gpurun_out/ab_c2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_c2_tests.log
tail -2 gpurun_out/ab_c2_tests.log
bash tools/gpu/abn.sh both "$@"
