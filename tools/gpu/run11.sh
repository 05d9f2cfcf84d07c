mkdir -p gpurun_out
(for o in sum sum,mean sum,cfg sum,mean,cfg; do echo "out=$o"; KB_OUT=$o timeout 120 python tools/kbench.py list 5; done) > gpurun_out/kbench17.log 2>&1
cat gpurun_out/kbench17.log
