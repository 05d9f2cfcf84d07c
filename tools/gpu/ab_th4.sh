mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "thief_bitexact or ties or config4_full or persistent or thief_invalid or scaleout" > gpurun_out/ab_th4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_th4_tests.log
tail -2 gpurun_out/ab_th4_tests.log
bash tools/gpu/abn.sh steepest "$@"
bash tools/gpu/abn.sh literal "$@"
