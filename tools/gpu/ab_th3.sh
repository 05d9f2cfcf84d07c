mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "thief or ties or config4 or config5 or place or window or gather or uniform" > gpurun_out/ab_th3_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_th3_tests.log
tail -2 gpurun_out/ab_th3_tests.log
bash tools/gpu/abn.sh steepest "$@"
bash tools/gpu/abn.sh literal "$@"
