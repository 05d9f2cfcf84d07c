for L in libekya_head.so libekya.so; do
 for m in steepest literal; do KBENCH_LIB=paper_2012_10557_b200/$L timeout 300 python tools/kbench.py $m 10; done
 for m in steepest literal; do KB_C5=1 KB_B=16384 KBENCH_LIB=paper_2012_10557_b200/$L timeout 300 python tools/kbench.py $m 5; done
done
timeout 900 python -m pytest tests -m gpu -q -x -k "thief or window or config4 or config5 or gather or ties or place or profile_output" 2>&1 | tail -2
