mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "grid or list or ties or config4 or uniform or window or place or profile_output" > gpurun_out/ab_gl_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_gl_tests.log
tail -2 gpurun_out/ab_gl_tests.log
bash tools/gpu/abn.sh grid "$@"
bash tools/gpu/abn.sh list "$@"
