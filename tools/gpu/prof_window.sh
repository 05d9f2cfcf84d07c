mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"window|thief" --csv --log-file gpurun_out/win_launches.csv python tools/win_driver.py > gpurun_out/win.log 2>&1
tail -2 gpurun_out/win.log
