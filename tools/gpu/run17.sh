mkdir -p gpurun_out
(for l in tools/variants/lib_base.so tools/variants/lib_nl5.so; do for k in grid list; do KBENCH_LIB=$l timeout 120 python tools/kbench.py $k 5; done; done) > gpurun_out/kbench26.log 2>&1
cat gpurun_out/kbench26.log
