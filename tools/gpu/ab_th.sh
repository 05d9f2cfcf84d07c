mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "thief or ties or config4 or config5 or place or window or gather" > gpurun_out/ab_th_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_th_tests.log
tail -2 gpurun_out/ab_th_tests.log
bash tools/gpu/abn.sh steepest tools/variants/vA.so tools/variants/vH.so tools/variants/vG.so
bash tools/gpu/abn.sh literal tools/variants/vA.so tools/variants/vH.so tools/variants/vG.so
KB_C5=1 KB_B=16384 bash tools/gpu/abn.sh steepest tools/variants/vA.so tools/variants/vG.so
