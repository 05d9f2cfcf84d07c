# thief A/B (parity, timings) + one ncu --set full capture per mode
bash tools/gpu/thief_ab.sh
mkdir -p gpurun_out/thief
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/thief/steep -f python tools/kbench.py steepest 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/thief/lit -f python tools/kbench.py literal 1 > /dev/null 2>&1
ls gpurun_out/thief
