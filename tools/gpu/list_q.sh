for a in "2048 256" "20000 100" "300 1"; do timeout 120 python tools/list_dbg.py $a 2>&1 | tail -1; done
timeout 600 python -m pytest tests -m gpu -q -x -k "list or config4 or ties" 2>&1 | tail -1
for i in 1 2; do timeout 300 python tools/kbench.py list 10; done
