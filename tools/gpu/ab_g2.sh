mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid or ties or config4" > gpurun_out/ab_g2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_g2_tests.log
tail -2 gpurun_out/ab_g2_tests.log
bash tools/gpu/abn.sh grid tools/variants/vA.so tools/variants/vE.so tools/variants/vF.so
