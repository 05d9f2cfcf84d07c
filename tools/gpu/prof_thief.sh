mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/steep2 -f python tools/kbench.py steepest 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:thief -s 2 -c 1 -o gpurun_out/lit2 -f python tools/kbench.py literal 1 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -2
