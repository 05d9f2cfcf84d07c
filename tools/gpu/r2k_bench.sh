# round-2 final evidence, part 2: the bench line (issue fractions from the refreshed instruction counts)
mkdir -p gpurun_out/r2k3
timeout 900 python bench.py > gpurun_out/r2k3/bench.json 2>gpurun_out/r2k3/bench.err; echo "bench rc=$?"
