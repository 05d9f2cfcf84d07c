mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prune_kernel -c 1 -o gpurun_out/prune1 -f python tools/prof_driver.py > gpurun_out/prune_prof.log 2>&1
tail -3 gpurun_out/prune_prof.log; ls gpurun_out/*.ncu-rep | tail -2
