timeout 120 python tools/list_dbg.py 20000 100 | tail -1
for r in 32 64 128 256; do echo "rpt=$r"; EKYA_LIST_RPT=$r timeout 120 python tools/list_dbg.py 3000 300 | tail -1; EKYA_LIST_RPT=$r timeout 300 python tools/kbench.py list 10; done
for a in 2 4 8; do echo "rpt=128 ahead=$a"; EKYA_LIST_RPT=128 EKYA_L2PF_AHEAD=$a timeout 300 python tools/kbench.py list 10; done
