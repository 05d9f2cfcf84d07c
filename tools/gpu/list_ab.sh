# LIST A/B: parity of every LIST test, kernel timings (list2 vs list_kernel via EKYA_LIST_V1), ncu capture
mkdir -p gpurun_out/list
python -c "import paper_2012_10557_b200.build as b; b.build()"
timeout 900 python -m pytest tests -m gpu -q -x -k "list or config4 or ties or smoke" > gpurun_out/list/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/list/tests.log
tail -3 gpurun_out/list/tests.log
timeout 300 python tools/kbench.py list 10 2>&1 | tee gpurun_out/list/kbench.txt
EKYA_LIST_V1=1 timeout 300 python tools/kbench.py list 10 2>&1 | tee -a gpurun_out/list/kbench.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:list -s 2 -c 1 -o gpurun_out/list/list2 -f python tools/kbench.py list 1 > gpurun_out/list/ncu.log 2>&1
tail -2 gpurun_out/list/ncu.log
