mkdir -p gpurun_out/list
timeout 120 python tools/list_dbg.py 20000 100 | tail -1
for m in 1 0; do echo "pf=$m"; EKYA_L2PF=$m timeout 300 python tools/kbench.py list 10; done
for a in 4 8 16 32 64; do echo "pf=2 ahead=$a"; EKYA_L2PF=2 EKYA_L2PF_AHEAD=$a timeout 300 python tools/kbench.py list 10; done
