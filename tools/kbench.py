"""Time one hot-path kernel in isolation (CUDA events, after warm-up) for quick A/B runs.
usage: python tools/kbench.py {cluster|radius|both|grid|list|steepest|literal} [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2012_10557_b200 import ekya  # noqa: E402

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
if os.environ.get("KBENCH_LIB"):   # A/B a variant build (tools only; the product loads LIB_PATH)
    ekya.load_library(os.environ["KBENCH_LIB"])
h = ekya.Handle(0)
w = bench.Workload(int(os.environ.get("KB_B", synth.CONFIG4.n_inst)), int(os.environ.get("KB_N", synth.CONFIG4.n_alloc)),
                   synth.CONFIG3.n_query)
if which in ("cluster", "radius", "both"):
    p = w.pcfg
    P = {}
    P["cur"] = torch.empty((w.Q, p.n_class), device=dev)
    P["hist"] = torch.empty((w.Q, p.n_hist, p.n_class), device=dev)
    P["hist_acc"] = torch.empty((w.Q, p.n_hist, p.n_gamma), device=dev)
    P["fallback"] = torch.empty((w.Q, p.n_gamma), device=dev)
    for q0 in range(0, w.Q, 2048):
        part = synth.profile_inputs(p, q0, min(w.Q, q0 + 2048), device=dev)
        for k in P:
            P[k][q0:q0 + 2048] = part[k]
    mode = ekya.PROFILE_CLUSTER if which == "cluster" else ekya.PROFILE_RADIUS
    if which == "both":
        fn = lambda: ekya.profile_estimate_both(h, P["cur"], P["hist"], P["hist_acc"], P["fallback"])
    else:
        fn = lambda: ekya.profile_estimate(h, P["cur"], P["hist"], P["hist_acc"], P["fallback"], mode=mode)
else:
    if os.environ.get("KB_C5"):   # config-5 shape (V = 100, U = 800)
        w.cfg = synth.SchedConfig(**{**synth.CONFIG5.__dict__, "n_inst": w.B})
        c = w.cfg
        w.args = (c.units, c.steal_units, c.unit_gpu_seconds, c.a_min)
    T = synth.sched_tables(w.cfg, 0, w.B, device=dev)
    args = w.args
    if which == "grid":
        grid = torch.empty((w.B, w.V, w.nc), dtype=torch.float32, device=dev)
        gcfg = torch.empty((w.B, w.V, w.nc), dtype=torch.uint8, device=dev)
        dims, tabs = ekya.dims_from(T, *args), ekya.make_tables(**T)
        fn = lambda: ekya.ekya_eval_allocations(h, dims, tabs, ekya.EVAL_GRID, out_grid=grid, out_grid_cfg=gcfg)
    elif which == "list":
        rows = torch.empty((w.B, w.N, w.J), dtype=torch.uint16, device=dev)
        for b0 in range(0, w.B, 1024):
            rows[b0:b0 + 1024] = synth.list_allocs(w.cfg, w.N, b0, min(w.B, b0 + 1024), device=dev)
        if os.environ.get("KB_OUT"):   # subset of LIST outputs, e.g. "sum" or "sum,mean"
            outs = os.environ["KB_OUT"].split(",")
            dims, tabs = ekya.dims_from(T, *args), ekya.make_tables(**T)
            ls = torch.empty((w.B, w.N), dtype=torch.uint64, device=dev)
            lm = torch.empty((w.B, w.N), dtype=torch.float32, device=dev) if "mean" in outs else None
            lc = torch.empty((w.B, w.N, w.V), dtype=torch.uint8, device=dev) if "cfg" in outs else None
            fn = lambda: ekya.ekya_eval_allocations(h, dims, tabs, ekya.EVAL_LIST, w.N, rows, ls, lm, lc)
        else:
            fn = lambda: ekya.eval_list(h, T, rows, *args)
    else:
        mode = ekya.THIEF_STEEPEST if which == "steepest" else ekya.THIEF_LITERAL
        fn = lambda: ekya.thief_schedule(h, T, *args, mode=mode)
for _ in range(2):
    fn()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
assert h.last_error() == 0
print(which, os.path.basename(os.environ.get("KBENCH_LIB", "libekya.so")), "ms", sorted(ts)[len(ts) // 2], "min", min(ts))
