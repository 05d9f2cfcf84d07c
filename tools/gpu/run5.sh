mkdir -p gpurun_out
for n in 32 256 1024 4096; do KB_N=$n timeout 120 python tools/kbench.py list 5; done > gpurun_out/kbench_listN.log 2>&1
cat gpurun_out/kbench_listN.log
