mkdir -p gpurun_out
(for bn in "65536 4096" "16384 16384" "4096 65536"; do set -- $bn; echo "B=$1 N=$2"; KB_B=$1 KB_N=$2 KB_OUT=sum,mean,cfg timeout 200 python tools/kbench.py list 5; done) > gpurun_out/kbench18.log 2>&1
cat gpurun_out/kbench18.log
