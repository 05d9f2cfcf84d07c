mkdir -p gpurun_out
(for l in tools/variants/lib_rs3.so tools/variants/lib_rs4.so; do KBENCH_LIB=$l timeout 120 python tools/kbench.py radius 5; done) > gpurun_out/kbench21.log 2>&1
cat gpurun_out/kbench21.log
