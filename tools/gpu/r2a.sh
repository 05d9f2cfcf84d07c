# round 2 first call: host info, measured FP32 SIMT peak, new parity tests
mkdir -p gpurun_out/r2a
(nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket") > gpurun_out/r2a/host.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader,nounits -lms 200 > gpurun_out/r2a/fp2_clocks.csv &
SMI=$!
./tools/micro/fp2 1965 > gpurun_out/r2a/fp2.log 2>&1
kill $SMI
python -c "import paper_2012_10557_b200.build as b; b.build()"
timeout 1500 python -m pytest tests -m gpu -q -x -k "bench_launch or config5_sample or config4_full" --durations=10 > gpurun_out/r2a/tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/tests.log
tail -3 gpurun_out/r2a/tests.log
