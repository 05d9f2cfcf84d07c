mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "list or ties or config4" > gpurun_out/ab_list_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_list_tests.log
tail -2 gpurun_out/ab_list_tests.log
bash tools/gpu/abn.sh list "$@"
