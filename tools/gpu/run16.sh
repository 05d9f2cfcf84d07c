mkdir -p gpurun_out
(for l in tools/variants/lib_lt1024.so tools/variants/lib_lt768.so tools/variants/lib_lt512.so; do KBENCH_LIB=$l timeout 120 python tools/kbench.py list 5; done) > gpurun_out/kbench22.log 2>&1
cat gpurun_out/kbench22.log
