for a in "2048 256" "20000 100" "300 1"; do timeout 120 python tools/list_dbg.py $a 2>&1 | tail -1; done
for m in 2 0; do echo "pf=$m"; EKYA_L2PF=$m timeout 300 python tools/kbench.py list 10; done
