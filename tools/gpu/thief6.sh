for ns in 2 4 8 16; do echo "NS=$ns"; for m in steepest literal; do EKYA_THIEF_NS=$ns KB_C5=1 KB_B=16384 timeout 300 python tools/kbench.py $m 5; done; done
