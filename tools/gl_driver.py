"""Launch the fused GRID + LIST mode (ekya_eval_allocations mode 2) of an A/B library once
or time it (tools only).  usage: KBENCH_LIB=lib.so python tools/gl_driver.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2012_10557_b200 import ekya  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
ekya.load_library(os.environ["KBENCH_LIB"])
h = ekya.Handle(0)
w = bench.Workload(65536, 4096, 0)
T = synth.sched_tables(w.cfg, 0, w.B, device=dev)
rows = bench.gen_list_rows(w, dev)
O = bench.Outputs(w, dev)
dims, tabs = ekya.dims_from(T, *w.args), ekya.make_tables(**T)
L = ekya.load_library()
P = lambda t: ctypes.c_void_p(t.data_ptr())
import ctypes  # noqa: E402
fn = lambda: L.ekya_eval_allocations(h.ptr, ctypes.byref(dims), ctypes.byref(tabs), 2, w.N, P(rows), P(O.lsum),
                                     P(O.lmean), P(O.lcfg), P(O.grid), P(O.grid_cfg), None)
for _ in range(2):
    assert fn() == 0
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("gridlist ms", sorted(ts)[len(ts) // 2])
