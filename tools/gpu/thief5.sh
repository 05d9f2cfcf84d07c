for L in libekya.so; do
 for m in steepest literal; do KBENCH_LIB=paper_2012_10557_b200/$L timeout 300 python tools/kbench.py $m 10; done
 for m in steepest literal; do KB_C5=1 KB_B=16384 KBENCH_LIB=paper_2012_10557_b200/$L timeout 300 python tools/kbench.py $m 5; done
done
