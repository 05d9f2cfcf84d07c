"""Launch each hot-path kernel a few times on a reduced-but-representative batch
(for ncu captures; timings taken under ncu are never bench values)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2012_10557_b200 import ekya  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-inst", type=int, default=65536)
ap.add_argument("--n-alloc", type=int, default=4096)
ap.add_argument("--n-query", type=int, default=65536)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
torch.cuda.set_device(0)
h = ekya.Handle(0)
w = bench.Workload(a.n_inst, a.n_alloc, a.n_query)
T, rows, P = bench.gen_device(w, torch.device("cuda", 0))
O = bench.Outputs(w, torch.device("cuda", 0))
for _ in range(a.reps):
    bench.run_step(ekya, h, w, T, rows, P, O)
torch.cuda.synchronize()
assert h.last_error() == 0
print("launches", h.launch_count())
