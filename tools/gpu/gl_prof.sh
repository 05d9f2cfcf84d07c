mkdir -p gpurun_out/gl
KBENCH_LIB=paper_2012_10557_b200/libekya_fused.so timeout 300 python tools/gl_driver.py 5
KBENCH_LIB=paper_2012_10557_b200/libekya_fused.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:list2 -s 2 -c 1 -o gpurun_out/gl/fused -f python tools/gl_driver.py 1 > gpurun_out/gl/ncu.log 2>&1
tail -1 gpurun_out/gl/ncu.log
