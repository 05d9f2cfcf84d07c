# round-2 final evidence, part 2: the bench line (issue fractions from the refreshed instruction counts)
mkdir -p gpurun_out/r2l
timeout 900 python bench.py > gpurun_out/r2l/bench.json 2>gpurun_out/r2l/bench.err; echo "bench rc=$?"
