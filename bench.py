#!/usr/bin/env python
"""bench.py -- Ekya thief-scheduler hot path on B200 (driver contract: one JSON line).

A step = one pass of the whole hot path over one batch:
  A1  ekya_profile_estimate_both on config 3 (65,536 Waymo-shaped queries, C=27,
      H=500, |Gamma|=18) in CLUSTER mode (BASELINE config 3: "5-cluster
      similarity estimate") and RADIUS mode (north star: distance threshold);
  A3  ekya_eval_allocations GRID and LIST (4,096 allocations per instance) on
      config 4 (65,536 Cityscapes-shaped 10-stream instances, |Gamma|=18,
      |Lambda|=5, U=80);
  A4-A6 ekya_thief_schedule STEEPEST and LITERAL on config 4.
Metric (BASELINE.json): scheduler allocations evaluated per second, where one
allocation = one (instance, stream, r_train, r_infer) split reduced over
Gamma x Lambda: GRID cells + LIST rows x V.  Thief schedules/s,
profile queries/s and per-kernel roofline fractions are reported under "rows".

--impl reference times the CPU oracle (tier rules: there is no reference
implementation) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "scheduler allocations evaluated/sec and thief schedules/sec; % HBM roofline"
UNIT = "allocations/s"

# The driver reads ONE JSON line from stdout.  Libraries write banners to fd 1 (NCCL prints
# its version line when NCCL_DEBUG is set in the environment), so fd 1 is pointed at stderr
# for the whole run and the JSON line goes to a private duplicate of the original stdout.
_JSON_OUT = None


def emit(line):
    global _JSON_OUT
    if _JSON_OUT is None:
        _JSON_OUT = sys.stdout
    _JSON_OUT.write(json.dumps(line) + "\n")
    _JSON_OUT.flush()


def _stdout_to_stderr():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def fp32_peak(sm_mhz):
    """Measured FP32 SIMT peak (TFLOP/s) scaled to `sm_mhz`, and its source."""
    p = os.path.join(ROOT, "profiles", "round2_fp32_peak.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        v = float(d["fp32_simt_tflops"]) * sm_mhz / float(d["sm_mhz"])
        return v, (f"measured: tools/micro/fp2.cu {d['fp32_simt_tflops']:.2f} TFLOP/s at {d['sm_mhz']:.0f} MHz "
                   f"(profiles/round2_fp32_peak.json), scaled to {sm_mhz:.0f} MHz")
    return 148 * 128 * sm_mhz * 1e6 / 1e12, f"derived: 148 SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz"


def inst_counts():
    """Warp instructions per launch of the issue-bound kernels from an ncu capture of the bench
    shapes (profiles/round2_inst.json: {kernel: {warp_inst_per_launch, units}})."""
    p = os.path.join(ROOT, "profiles", "round2_inst.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured", d
    return 6650.0, "fallback", {}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------
class Workload:
    def __init__(self, n_inst, n_alloc, n_query, inst_offset=0, query_offset=0):
        self.cfg = synth.SchedConfig(**{**synth.CONFIG4.__dict__, "n_inst": inst_offset + n_inst,
                                        "n_alloc": n_alloc})
        self.pcfg = synth.ProfileConfig(**{**synth.CONFIG3.__dict__, "n_query": query_offset + n_query})
        self.B, self.N, self.Q = n_inst, n_alloc, n_query
        self.i0, self.q0 = inst_offset, query_offset
        c = self.cfg
        self.V, self.J, self.U = c.n_streams, 2 * c.n_streams, c.units
        self.nc = (c.units + 1) * (c.units + 2) // 2
        self.args = (c.units, c.steal_units, c.unit_gpu_seconds, c.a_min)

    # units of the metric in one step
    def allocations(self):
        return self.B * self.V * self.nc + self.B * self.N * self.V

    # algorithmic bytes per launch
    def table_bytes(self):
        c = self.cfg
        return self.B * self.V * (4 + 8 * c.n_gamma + 6 * c.n_lambda)

    def grid_bytes(self):
        return self.table_bytes() + self.B * self.V * self.nc * 5

    def list_bytes(self):
        return self.table_bytes() + self.B * self.N * (2 * self.J + 8 + 4 + self.V)

    def profile_bytes(self):
        p = self.pcfg
        return self.Q * (4 * (p.n_hist * (p.n_class + p.n_gamma) + p.n_class + p.n_gamma) + 8 * p.n_gamma)

    def thief_bytes(self):
        return self.table_bytes() + self.B * (2 * self.J + self.V + 16)


def gen_list_rows(w: Workload, dev):
    """LIST allocation rows of the step (device generation in 1,024-instance chunks)."""
    rows = torch.empty((w.B, w.N, w.J), dtype=torch.uint16, device=dev)
    ch = 1024
    for b0 in range(0, w.B, ch):
        b1 = min(w.B, b0 + ch)
        rows[b0:b1] = synth.list_allocs(w.cfg, w.N, w.i0 + b0, w.i0 + b1, device=dev)
    return rows


def gen_device(w: Workload, dev):
    """Generate the batch on the device in chunks (bit-identical to CPU generation)."""
    T = synth.sched_tables(w.cfg, w.i0, w.i0 + w.B, device=dev)
    rows = gen_list_rows(w, dev)
    p = w.pcfg
    P = {"cur": torch.empty((w.Q, p.n_class), device=dev),
         "hist": torch.empty((w.Q, p.n_hist, p.n_class), device=dev),
         "hist_acc": torch.empty((w.Q, p.n_hist, p.n_gamma), device=dev),
         "fallback": torch.empty((w.Q, p.n_gamma), device=dev)}
    ch = 2048
    for q0 in range(0, w.Q, ch):
        q1 = min(w.Q, q0 + ch)
        part = synth.profile_inputs(p, w.q0 + q0, w.q0 + q1, device=dev)
        for k in P:
            P[k][q0:q1] = part[k]
        del part
    torch.cuda.synchronize()
    return T, rows, P


class Outputs:
    def __init__(self, w: Workload, dev):
        B, V, J, N, Q, G = w.B, w.V, w.J, w.N, w.Q, w.pcfg.n_gamma
        self.grid = torch.empty((B, V, w.nc), dtype=torch.float32, device=dev)
        self.grid_cfg = torch.empty((B, V, w.nc), dtype=torch.uint8, device=dev)
        self.lsum = torch.empty((B, N), dtype=torch.uint64, device=dev)
        self.lmean = torch.empty((B, N), dtype=torch.float32, device=dev)
        self.lcfg = torch.empty((B, N, V), dtype=torch.uint8, device=dev)
        # decision records (one contiguous buffer per mode: gathered to the root for N > 1)
        from paper_2012_10557_b200 import shard
        self.rec_bytes = shard.record_bytes(B, V)
        self.dec = []
        for _ in range(2):
            buf = torch.empty(self.rec_bytes, dtype=torch.uint8, device=dev)
            self.dec.append(dict(buf=buf, **shard.record_views(buf, B, V)))
        self.est = [torch.empty((Q, G), dtype=torch.float32, device=dev) for _ in range(2)]
        self.n = [torch.empty((Q, G), dtype=torch.int32, device=dev) for _ in range(2)]


def run_step(ek, h, w, T, rows, P, O, timer=None):
    """One pass of the whole hot path.  Returns nothing; all work on the current stream."""
    dims = ek.dims_from(T, *w.args)
    tabs = ek.make_tables(**T)
    p = w.pcfg
    steps = []
    if os.environ.get("EKYA_BENCH_PROFILE_UNFUSED"):   # A/B: the two modes as separate launches
        steps += [
            ("profile_cluster", lambda: ek.ekya_profile_estimate(
                h, ek.ProfileDims(w.Q, p.n_hist, p.n_class, p.n_gamma, ek.PROFILE_CLUSTER, p.tau, p.k, p.max_iter),
                P["cur"], P["hist"], P["hist_acc"], P["fallback"], O.est[1], O.n[1])),
            ("profile_radius", lambda: ek.ekya_profile_estimate(
                h, ek.ProfileDims(w.Q, p.n_hist, p.n_class, p.n_gamma, ek.PROFILE_RADIUS, p.tau, p.k, p.max_iter),
                P["cur"], P["hist"], P["hist_acc"], P["fallback"], O.est[0], O.n[0]))]
    else:
        # A1: both estimates (RADIUS tau = 0.2 and CLUSTER k = 5) from ONE pass over each query's
        # history tile (ekya_profile_estimate_both)
        steps += [("profile", lambda: ek.ekya_profile_estimate_both(
            h, ek.ProfileDims(w.Q, p.n_hist, p.n_class, p.n_gamma, ek.PROFILE_CLUSTER, p.tau, p.k, p.max_iter),
            P["cur"], P["hist"], P["hist_acc"], P["fallback"], O.est[0], O.n[0], O.est[1], O.n[1]))]
    steps += [
        ("eval_grid", lambda: ek.ekya_eval_allocations(h, dims, tabs, ek.EVAL_GRID, out_grid=O.grid,
                                                       out_grid_cfg=O.grid_cfg)),
        ("eval_list", lambda: ek.ekya_eval_allocations(h, dims, tabs, ek.EVAL_LIST, w.N, rows, O.lsum,
                                                       O.lmean, O.lcfg)),
        ("thief_steepest", lambda: ek.ekya_thief_schedule(h, dims, tabs, ek.THIEF_STEEPEST, O.dec[0]["alloc"],
                                                          O.dec[0]["cfg"], O.dec[0]["sum"], O.dec[0]["mean"],
                                                          O.dec[0]["steps"])),
        ("thief_literal", lambda: ek.ekya_thief_schedule(h, dims, tabs, ek.THIEF_LITERAL, O.dec[1]["alloc"],
                                                         O.dec[1]["cfg"], O.dec[1]["sum"], O.dec[1]["mean"],
                                                         O.dec[1]["steps"])),
    ]
    for name, fn in steps:
        if timer is not None:
            timer.start(name)
        fn()
        if timer is not None:
            timer.stop(name)


class KernelTimer:
    """CUDA events on the launching (current) stream around each launch."""

    def __init__(self):
        self.ev = {}

    def start(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev.setdefault(name, []).append([e, None])

    def stop(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.ev[name][-1][1] = e

    def totals_ms(self):
        return {k: sum(a.elapsed_time(b) for a, b in v) for k, v in self.ev.items()}

    def launches_ms(self):
        return {k: [a.elapsed_time(b) for a, b in v] for k, v in self.ev.items()}


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.first = threading.Event()

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self.first.set()

    def wait_first(self, timeout=10.0):
        """Block until the sampler has produced its first line (nvidia-smi can take
        over a second to start), so the timed region is covered from its start."""
        if self.proc:
            self.first.wait(timeout)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_threads():
    import oracle
    return oracle.host_threads()


def ref_sizes(args):
    """Bounded oracle sample: 256 config-4 instances + 128 config-3 queries per host thread
    (about 3-4 s of wall time per sample on any core count), unless given."""
    t = oracle_threads()
    return (args.ref_inst or min(65536, 256 * t)), (args.ref_query or min(65536, 128 * t))


def oracle_sample(n_inst, n_query):
    """One bounded sample of the same workload through the oracle, its independent instances
    and queries spread over a thread pool of all host cores (the per-instance code is the
    plain single-threaded oracle).  Returns (seconds, allocations evaluated, description,
    threads)."""
    from concurrent.futures import ThreadPoolExecutor
    import oracle
    threads = oracle.host_threads()
    w = Workload(n_inst, synth.CONFIG4.n_alloc, n_query)
    T = synth.sched_tables(w.cfg, 0, n_inst)
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *w.args)
    rows = synth.list_allocs(w.cfg, w.N, 0, n_inst).numpy()
    P = {k: v.numpy() for k, v in synth.profile_inputs(w.pcfg, 0, n_query).items()}
    qb = np.linspace(0, n_query, min(n_query, 4 * threads) + 1).astype(np.int64)
    blocks = [(a, b) for a, b in zip(qb[:-1], qb[1:]) if b > a]
    oracle.lib()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for mode in (oracle.CLUSTER, oracle.RADIUS):
            list(ex.map(lambda ab: oracle.profile(P["cur"][ab[0]:ab[1]], P["hist"][ab[0]:ab[1]],
                                                  P["hist_acc"][ab[0]:ab[1]], P["fallback"][ab[0]:ab[1]],
                                                  mode=mode), blocks))
    oracle.per_instance_parallel(oracle.eval_grid, inst, threads=threads)
    oracle.per_instance_parallel(oracle.eval_list, inst, rows, threads=threads)
    oracle.per_instance_parallel(oracle.thief, inst, oracle.STEEPEST, threads=threads)
    oracle.per_instance_parallel(oracle.thief, inst, oracle.LITERAL, threads=threads)
    dt = time.perf_counter() - t0
    desc = (f"{n_inst} of 65536 config-4 instances (GRID, LIST x4096, thief STEEPEST+LITERAL) + "
            f"{n_query} of 65536 config-3 queries (CLUSTER+RADIUS); oracle on a pool of {threads} threads "
            f"(all host cores), instances/queries split across them")
    return dt, w.allocations(), desc, threads


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    oracle.build()
    ni, nq = ref_sizes(args)
    for _ in range(args.warmup):
        oracle_sample(ni, nq)
    ts, units = [], 0
    desc, threads = "", 1
    for _ in range(args.steps):
        dt, units, desc, threads = oracle_sample(ni, nq)
        ts.append(dt)
    tot = float(sum(ts))
    value = units * args.steps / tot
    w = Workload(synth.CONFIG4.n_inst, synth.CONFIG4.n_alloc, synth.CONFIG3.n_query)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_block(w, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def config_block(w, args):
    return {"workload": "config4 (65,536 x 10-stream Cityscapes-shaped instances, |Gamma|=18, |Lambda|=5, "
                        "U=80, Delta=0.1 GPU, GRID + LIST(4096/inst) + thief STEEPEST+LITERAL) + config3 "
                        "(65,536 Waymo-shaped profiler queries, C=27, H=500, |Gamma|=18, CLUSTER k=5 + RADIUS "
                        "tau=0.2)",
            "instances_per_gpu": w.B, "streams": w.V, "units": w.U, "list_rows_per_instance": w.N,
            "profile_queries_per_gpu": w.Q,
            "l2": "not flushed: every step streams > 126 MB (GRID writes 11 GB, profile reads 5.9 GB)",
            "parallelism": f"instance sharding x{args.gpus} + NCCL gather of decisions" if args.gpus > 1
            else "single GPU"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    from paper_2012_10557_b200 import ekya as ek
    ek.load_library()          # fails loudly if the CUDA library is missing
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    h = ek.Handle(local_rank)
    # the decision gather runs through an NCCL communicator at every N (one rank at N = 1)
    uid = [ek.ekya_comm_unique_id() if rank == 0 else None]
    if world > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(uid, src=0)
    ek.ekya_comm_init(h, uid[0], world, rank)
    comm_nranks, comm_rank = ek.ekya_comm_info(h)
    assert comm_nranks == world and comm_rank == rank, "NCCL communicator does not match the launch"
    w = Workload(args.n_inst, args.n_alloc, args.n_query, inst_offset=rank * args.n_inst,
                 query_offset=rank * args.n_query)
    T, rows, P = gen_device(w, dev)
    O = Outputs(w, dev)
    root_buf = [torch.empty(world * O.rec_bytes, dtype=torch.uint8, device=dev) if rank == 0 else None
                for _ in range(2)]

    def step(timer=None):
        run_step(ek, h, w, T, rows, P, O, timer)
        # final gather of both modes' decision records to rank 0 (ncclGather; 66 B/instance)
        if timer is not None:
            timer.start("gather")
        for m in range(2):
            ek.ekya_gather_decisions(h, O.dec[m]["buf"], root_buf[m], root=0)
        if timer is not None:
            timer.stop("gather")

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert h.last_error() == 0, "device reported a data error"

    # ---- device-resident timed region ----
    timer = KernelTimer()
    barrier()
    torch.cuda.synchronize()
    c0 = h.counters()
    with ClockSampler(local_rank) as clk:
        clk.wait_first()           # the sampler is running before the timed region starts
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            step(timer)
        t1.record()
        torch.cuda.synchronize()
    barrier()
    c1 = h.counters()
    launches = c1["launches"] - c0["launches"]
    lloyd_passes = c1["lloyd_passes"] - c0["lloyd_passes"]
    ms = t0.elapsed_time(t1)
    per = timer.totals_ms()
    per_launch = timer.launches_ms()
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())

    # ---- end-to-end through the public API with host buffers ----
    e2e = None
    if args.e2e_steps > 0:
        e2e = run_e2e(ek, h, w, T, rows, P, O, args, world)

    c5 = run_config5(ek, h, dev, args, rank, world) if args.c5_inst > 0 else None
    context = run_context(ek, h, dev, args) if rank == 0 and args.context else None
    if context is not None:
        context.update(run_next1(ek, h, w, T, O, dev))
        context.update(run_next2(ek, h, w, dev))
        context.update(run_next3(ek, h, w, T, O, dev))
        context.update(run_next3_prune(ek, h, w, T, P))
        context.update(run_next4(ek, h, w, O, dev))
    if rank != 0:
        return
    peak, peak_kind, mp = measured_peaks()
    clocks = clk.summary()
    sm_mhz = float(clocks.get("sm_mhz") or mp.get("sm_max_mhz", 1965.0))
    # FP32 SIMT peak for the ALU-bound CLUSTER kernel: MEASURED (tools/micro/fp2.cu: FADD /
    # FMUL / FADD2 / FMUL2 streams, profiles/round2_fp32_peak.json) at its clock, scaled to
    # the SM clock sampled during the timed region; one flop per FSUB/FMUL/FADD (the
    # arithmetic contract allows no FMA)
    alu_peak, alu_src = fp32_peak(sm_mhz)
    insts = inst_counts()
    total_units = w.allocations() * world * args.steps
    value = total_units / (ms / 1000.0)
    rows_out = {}
    bytes_of = {"eval_grid": w.grid_bytes(), "eval_list": w.list_bytes(), "profile_radius": w.profile_bytes(),
                "profile_cluster": w.profile_bytes(), "profile": w.profile_bytes(), "thief_steepest": w.thief_bytes(),
                "thief_literal": w.thief_bytes()}
    pc = w.pcfg
    cluster_flops = lloyd_passes / max(1, args.steps) * pc.n_hist * pc.k * pc.n_class * 3
    roof = {}
    for k, t in per.items():
        avg = t / args.steps
        r = {"ms_per_launch": avg, "share": t / ms}
        if per_launch.get(k):   # median and best of the timed launches as well
            r["ms_median"] = float(np.median(per_launch[k]))
            r["ms_best"] = float(min(per_launch[k]))
        if k in bytes_of:
            gbs = bytes_of[k] / (avg / 1000.0) / 1e9
            r["algorithmic_gb_per_s"] = gbs
            r["hbm_frac"] = gbs / peak
            roof[k] = {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                       "peak_source": peak_kind, "algorithmic_bytes_per_launch": bytes_of[k]}
        if k in ("profile_cluster", "profile"):
            # CLUSTER's Lloyd distances (+ the fused RADIUS distances: one per window, H C 3 flop)
            fl = cluster_flops + (w.Q * pc.n_hist * pc.n_class * 3 if k == "profile" else 0)
            tfs = fl / (avg / 1000.0) / 1e12
            r["algorithmic_tflop_per_s"] = tfs
            r["alu_frac"] = tfs / alu_peak
            r["lloyd_passes_per_query"] = lloyd_passes / max(1, args.steps) / w.Q
            roof[k] = {"bound": "alu", "achieved": tfs, "peak": alu_peak, "unit": "TFLOP/s", "frac": tfs / alu_peak,
                       "peak_source": alu_src, "algorithmic_flops_per_launch": fl}
        if k in insts:
            # issue-slot utilisation: warp instructions per launch (ncu sm__inst_executed.sum of the
            # same launch, profiles/round2_inst.json) / (4 issue slots x 148 SMs x clock x time)
            wi = insts[k]["warp_inst_per_launch"] * w.B / insts[k]["units"]
            r["warp_inst_per_unit"] = insts[k]["warp_inst_per_launch"] / insts[k]["units"]
            r["issue_frac"] = wi / (avg / 1000.0) / (4 * 148 * sm_mhz * 1e6) if not k.startswith("profile") else \
                insts[k]["warp_inst_per_launch"] * w.Q / insts[k]["units"] / (avg / 1000.0) / (4 * 148 * sm_mhz * 1e6)
        if k.startswith("thief"):
            r["schedules_per_s"] = w.B * world / (avg / 1000.0)
            r.pop("hbm_frac", None)      # issue-bound: the HBM fraction says nothing here
            r.pop("algorithmic_gb_per_s", None)
        if k.startswith("profile"):
            r["queries_per_s"] = w.Q * world / (avg / 1000.0)
        if k.startswith("eval_grid"):
            r["cells_per_s"] = w.B * w.V * w.nc * world / (avg / 1000.0)
            # the north star's tuple count, cells x (|Gamma| + 1) x |Lambda| --
            # DERIVED (the (gamma, lambda) enumeration the per-stream tables avoid), not work done
            r["tuple_equiv_per_s_derived"] = r["cells_per_s"] * (T["cost"].shape[2] + 1) * T["lam_factor"].shape[2]
        if k.endswith("list"):
            r["allocation_vectors_per_s"] = w.B * w.N * world / (avg / 1000.0)
        rows_out[k] = r
    dom = max((k for k in per if k in roof), key=lambda k: per[k])
    roofline = dict(roof[dom])
    roofline["kernel"] = dom
    roofline["traffic"] = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            roofline["traffic"] = json.load(f).get(dom)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded counter-based generator, paper shapes)",
        "config": config_block(w, args),
        "roofline": roofline,
        "rows": rows_out,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if context is not None:
        line["context"] = context
    if c5 is not None:
        line.setdefault("context", {}).update(c5)
    line["comm"] = {"backend": "nccl", "nranks": comm_nranks, "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                    "gather": "ncclGather of the decision records to rank 0 (ekya_gather_decisions)"}
    if args.cpu_baseline and world == 1:
        import oracle
        oracle.build()
        dt, units, desc, threads = oracle_sample(*ref_sizes(args))
        line["cpu_baseline"] = {"value": units / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
                                "sample": desc, "seconds": dt, "nproc": os.cpu_count()}
        # NEXT-4 placement: the oracle on 4,096 of the step's STEEPEST decisions (one thread)
        sample = O.dec[0]["alloc"][:4096].cpu().numpy()
        t0 = time.perf_counter()
        oracle.place(sample, w.U, 8)
        line["cpu_baseline"]["next4_placement_instances_per_s"] = sample.shape[0] / (time.perf_counter() - t0)
    emit(line)


def _time_ms(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_next3(ek, h, w, T, O, dev):
    """SURVEY 8(f) NEXT-3 beside the step: the uniform baseline (even split, each stream's
    highest-accuracy config) on the step's 65,536 config-4 instances -- its mean
    objective against the two thieves' (the uniform <= thief sandwich at scale) -- and the
    Pareto frontier of every stream's 18 configurations."""
    dims, tabs = ek.dims_from(T, *w.args), ek.make_tables(**T)
    B, V = w.B, w.V
    ua = torch.empty((B, 2 * V), dtype=torch.uint16, device=dev)
    uc = torch.empty((B, V), dtype=torch.uint8, device=dev)
    us = torch.empty((B,), dtype=torch.uint64, device=dev)
    um = torch.empty((B,), dtype=torch.float32, device=dev)
    ms_u = _time_ms(lambda: ek.ekya_uniform_schedule(h, dims, tabs, -1, 0.5, ua, uc, us, um))
    mask = torch.empty((B, V), dtype=torch.uint32, device=dev)
    ms_p = _time_ms(lambda: ek.ekya_pareto(h, T["cost"], T["post"], mask))
    assert h.last_error() == 0
    peak, _, _ = measured_peaks()
    G = T["cost"].shape[2]
    bytes_u = w.table_bytes() + B * (4 * V + V + 8 + 4)
    bytes_p = B * V * (8 * G + 4)
    m = mask.cpu().numpy().view(np.uint32)
    frontier = float(np.unpackbits(m.view(np.uint8)).sum()) / m.size
    return {"next3_uniform": {"instances": B, "ms": ms_u, "instances_per_s": B / (ms_u / 1000.0),
                              "hbm_frac": bytes_u / (ms_u / 1000.0) / 1e9 / peak,
                              "mean_objective_uniform": float(um.mean()),
                              "mean_objective_thief_steepest": float(O.dec[0]["mean"].mean()),
                              "mean_objective_thief_literal": float(O.dec[1]["mean"].mean()),
                              "uniform_le_thief_all": bool((us.cpu().numpy().view(np.uint64) <=
                                                            O.dec[1]["sum"].cpu().numpy().view(np.uint64)).all())},
            "next3_pareto": {"sets": B * V, "configs": G, "ms": ms_p, "sets_per_s": B * V / (ms_p / 1000.0),
                             "hbm_frac": bytes_p / (ms_p / 1000.0) / 1e9 / peak,
                             "mean_frontier_size": frontier}}


def run_next3_prune(ek, h, w, T, P):
    """SURVEY 8(f) NEXT-3's pruning beside the step (readings PN1-PN3): the
    step's 65,536 config-3 profiler histories (500 windows x 18 configs) against the config-4
    tables' costs of the first 65,536 streams, margin 0.05."""
    Q, H, G = P["hist_acc"].shape
    cost = T["cost"].reshape(-1, T["cost"].shape[-1])[:Q, :G].contiguous()
    keep = torch.empty((Q,), dtype=torch.uint32, device=cost.device)
    ms = _time_ms(lambda: ek.ekya_prune_configs(h, cost, P["hist_acc"], 0.05, keep))
    assert h.last_error() == 0
    peak, _, _ = measured_peaks()
    nbytes = Q * (H * G * 4 + G * 4 + 4)
    k = keep.cpu().numpy().view(np.uint32)
    kept = float(np.unpackbits(k.view(np.uint8)).sum()) / k.size
    return {"next3_prune": {"streams": Q, "windows": H, "configs": G, "margin": 0.05, "ms": ms,
                            "streams_per_s": Q / (ms / 1000.0),
                            "hbm_frac": nbytes / (ms / 1000.0) / 1e9 / peak,
                            "mean_configs_kept": kept}}


def run_next1(ek, h, w, T, O, dev):
    """SURVEY 8(f) NEXT-1 beside the step: the window timeline with the thief re-invoked at
    every retraining completion, over the step's 65,536 config-4 instances (STEEPEST):
    realized window-average accuracy vs the thief's t = 0 estimate."""
    dims, tabs = ek.dims_from(T, *w.args), ek.make_tables(**T)
    B, V = w.B, w.V
    ws = torch.empty((ek.ekya_window_workspace_bytes(dims),), dtype=torch.uint8, device=dev)
    avg = torch.empty((B,), dtype=torch.float32, device=dev)
    ev = torch.empty((B,), dtype=torch.uint32, device=dev)
    done = torch.empty((B, V), dtype=torch.float32, device=dev)
    ms = _time_ms(lambda: ek.ekya_window_schedule(h, dims, tabs, ek.THIEF_STEEPEST, ws, avg, ev, done), reps=2)
    assert h.last_error() == 0
    return {"next1_window": {"instances": B, "ms": ms, "instances_per_s": B / (ms / 1000.0),
                             "thief_invocations_per_instance": float(ev.cpu().numpy().view(np.uint32).mean()),
                             "mean_realized_accuracy": float(avg.mean()),
                             "mean_t0_estimate": float(O.dec[0]["mean"].mean()),
                             "streams_retrained_frac": float((done < 1).float().mean())}}


def run_next2(ek, h, w, dev):
    """SURVEY 8(f) NEXT-2 beside the step: the micro-profiler curve fit for every
    (stream, config) of 65,536 config-4 streams (5 profiled epochs, "say, 5"),
    extrapolated to 30 epochs -- the `post` input of a table."""
    S, P = w.B * w.cfg.n_gamma, 5
    g = torch.Generator(device="cpu").manual_seed(9)
    k = torch.arange(1, P + 1, dtype=torch.float64)
    b0 = 0.1 + 1.9 * torch.rand(S, 1, generator=g, dtype=torch.float64)
    b1 = 0.8 + 2.2 * torch.rand(S, 1, generator=g, dtype=torch.float64)
    b2 = 0.3 * torch.rand(S, 1, generator=g, dtype=torch.float64)
    a = (1.0 - (1.0 / (b0 * k + b1) + b2) + 0.02 * torch.randn(S, P, generator=g, dtype=torch.float64))
    acc = a.clamp(0, 1).to(torch.float32).to(dev)
    K = torch.full((S,), 30, dtype=torch.int32, device=dev)
    pred = torch.empty((S,), dtype=torch.float32, device=dev)
    ms = _time_ms(lambda: ek.ekya_curve_fit(h, acc, K, pred), reps=3)
    assert h.last_error() == 0
    # algorithmic work per set: 257 grid points x (the 2x2 NNLS + residuals over 5 points)
    flops = S * 257 * (2 * P + 10 + 4 * P)
    peak_alu = fp32_peak(1965.0)[0]
    return {"next2_curve_fit": {"sets": S, "points": P, "ms": ms, "sets_per_s": S / (ms / 1000.0),
                                "alu_frac": flops / (ms / 1000.0) / 1e12 / peak_alu}}


def run_next4(ek, h, w, O, dev):
    """SURVEY 8(f) NEXT-4 beside the step: placement of the step's STEEPEST decisions
    (65,536 instances x 20 jobs) onto the 8 GPUs of config 4 (0.1 GPU per unit), and
    checkpoint decisions for one (stream, time) point per stream."""
    gpus = 8
    alloc = O.dec[0]["alloc"]
    B, J = alloc.shape
    P = J + gpus
    pj = torch.empty((B, P), dtype=torch.uint16, device=dev)
    pq = torch.empty((B, P), dtype=torch.uint32, device=dev)
    pg = torch.empty((B, P), dtype=torch.int16, device=dev)
    npc = torch.empty((B,), dtype=torch.uint16, device=dev)
    load = torch.empty((B, gpus), dtype=torch.uint32, device=dev)
    ms_p = _time_ms(lambda: ek.ekya_place(h, w.U, gpus, alloc, pj, pq, pg, npc, load))
    n = B * w.V
    g = torch.Generator(device="cpu").manual_seed(5)
    T = torch.full((n,), 200.0)
    tau = T * torch.rand(n, generator=g)
    t = tau * torch.rand(n, generator=g)
    a, ast, A = (torch.rand(n, generator=g) for _ in range(3))
    dl = 5.0 * torch.rand(n, generator=g)
    xs = [x.to(dev) for x in (tau, t, T, a, ast, A, dl)]
    out = torch.empty((n,), dtype=torch.uint8, device=dev)
    ms_c = _time_ms(lambda: ek.ekya_checkpoint_decide(h, *xs, out))
    assert h.last_error() == 0
    peak, _, _ = measured_peaks()
    bytes_p = B * (2 * J + P * 8 + 2 + 4 * gpus)     # alloc in; pieces, count, loads out
    bytes_c = n * (7 * 4 + 1)
    res = {"next4_placement": {"instances": B, "jobs": J, "gpus": gpus, "ms": ms_p,
                               "instances_per_s": B / (ms_p / 1000.0),
                               "hbm_frac": bytes_p / (ms_p / 1000.0) / 1e9 / peak},
           "next4_checkpoint": {"points": n, "ms": ms_c, "decisions_per_s": n / (ms_c / 1000.0),
                                "hbm_frac": bytes_c / (ms_c / 1000.0) / 1e9 / peak}}
    return res


def run_context(ek, h, dev, args):
    """Context numbers beside the step (not part of `value`): single-instance thief
    latency at config 2 (the paper's 9.4 s for 10 streams x 8 GPUs x 18 configs,
    P:1294, was a host-side scheduler on other hardware) and config-5-shaped
    (V=100, U=800) thief throughput on one GPU."""
    out = {}
    c2 = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": 1})
    T2 = synth.sched_tables(c2, device=dev)
    a2 = (c2.units, c2.steal_units, c2.unit_gpu_seconds, c2.a_min)
    for name, mode in (("steepest", ek.THIEF_STEEPEST), ("literal", ek.THIEF_LITERAL)):
        for _ in range(3):
            ek.thief_schedule(h, T2, *a2, mode=mode)
        ts = []
        for _ in range(20):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ek.thief_schedule(h, T2, *a2, mode=mode)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[f"config2_single_instance_thief_{name}_ms"] = float(np.median(ts))
    out["paper_thief_latency_s"] = {"value": 9.4, "cite": "P:1294, 10 streams x 8 GPUs x 18 configs, "
                                    "host-side scheduler (PyTorch + Ray on AWS p3, P:1321)"}
    n5 = args.context_v100
    c5 = synth.SchedConfig(**{**synth.CONFIG5.__dict__, "n_inst": n5})
    T5 = synth.sched_tables(c5, device=dev)
    a5 = (c5.units, c5.steal_units, c5.unit_gpu_seconds, c5.a_min)
    for name, mode in (("steepest", ek.THIEF_STEEPEST), ("literal", ek.THIEF_LITERAL)):
        ek.thief_schedule(h, T5, *a5, mode=mode)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ek.thief_schedule(h, T5, *a5, mode=mode)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        out[f"config5_shape_thief_{name}"] = {"instances": n5, "ms": ms, "schedules_per_s": n5 / (ms / 1000.0)}
    return out


def run_config5(ek, h, dev, args, rank, world):
    """BASELINE config 5: 100 streams x 1M instances (V = 100, |Gamma| = 18, |Lambda| = 5,
    U = 800) sharded over the ranks (rank r owns shard_range(1M, N, r), generated locally from
    global instance ids), thief STEEPEST + LITERAL per chunk, and the decision records (516 B
    per instance and mode) gathered to rank 0 chunk by chunk on a second stream while the next
    chunk computes.  Runs on every rank (the gathers are collective); timed
    with CUDA events on the compute stream after it waits for the last gather, max over
    ranks.  Also timed: the same pass without gathers and the gathers alone (overlap).
    Rank 0 reports a SHA-256 of the gathered decisions in global instance order, which is
    the same at every N when the root buffer is byte-identical to the one-GPU run."""
    import hashlib
    from paper_2012_10557_b200 import shard
    total = args.c5_inst
    cfg = synth.SchedConfig(**{**synth.CONFIG5.__dict__, "n_inst": total})
    lo, hi = shard.shard_range(total, world, rank)
    B, V = hi - lo, cfg.n_streams
    parts = [synth.sched_tables(cfg, b0, min(hi, b0 + 16384), device=dev) for b0 in range(lo, hi, 16384)]
    T = {k: torch.cat([p[k] for p in parts]) for k in parts[0]} if parts else None
    del parts
    torch.cuda.synchronize()
    L = shard.RecordLayout(total, world, V, args.c5_chunks)
    bufs = [torch.zeros(L.rank_bytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    roots = [torch.zeros(L.root_bytes, dtype=torch.uint8, device=dev) if rank == 0 else None for _ in range(2)]
    a5 = (cfg.units, cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)
    chunks = []
    for c in range(L.n_chunks):
        b0, b1 = L.chunk_range(rank, c)
        Tc = {k: v[b0:b1] for k, v in T.items()}
        chunks.append((ek.dims_from(Tc, *a5), ek.make_tables(**Tc), [L.views(bufs[m], rank, c) for m in range(2)], Tc))
    comp = torch.cuda.current_stream()
    comm = torch.cuda.Stream()

    def one_pass(gather=True, compute=True):
        for c in range(L.n_chunks):
            if compute:
                dims, tabs, vs, _ = chunks[c]
                for m, mode in enumerate((ek.THIEF_STEEPEST, ek.THIEF_LITERAL)):
                    v = vs[m]
                    if dims.n_inst:
                        ek.ekya_thief_schedule(h, dims, tabs, mode, v["alloc"], v["cfg"], v["sum"], v["mean"],
                                               v["steps"])
            if gather:
                e = torch.cuda.Event()
                e.record(comp)
                comm.wait_event(e)
                for m in range(2):
                    ek.ekya_gather_decisions(h, L.local_chunk(bufs[m], c),
                                             L.root_chunk(roots[m], c) if rank == 0 else None, root=0, stream=comm)
        comp.wait_stream(comm)

    def timed(**kw):
        one_pass(**kw)
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(comp)
        comm.wait_event(t0)
        for _ in range(args.c5_reps):
            one_pass(**kw)
        t1.record(comp)
        torch.cuda.synchronize()
        ms = torch.tensor([t0.elapsed_time(t1) / args.c5_reps], dtype=torch.float64, device=dev)
        if world > 1:
            import torch.distributed as dist
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item())

    ms_all = timed()
    assert h.last_error() == 0
    digest = None
    if rank == 0:
        hsh = hashlib.sha256()
        for m in range(2):
            g = L.unpack(roots[m])
            for k in ("alloc", "cfg", "sum", "mean", "steps"):
                hsh.update(g[k].contiguous().view(torch.uint8).cpu().numpy().tobytes())
        digest = hsh.hexdigest()
    ms_comp = timed(gather=False)
    ms_gather = timed(compute=False)
    rec = L.chunk_bytes * L.n_chunks
    res = {"config5": {
        "workload": "BASELINE config 5: 100 streams x 1M instances, |Gamma|=18, |Lambda|=5, U=800 (Delta=0.1 GPU of "
                    "80 GPUs), sharded over the ranks; thief STEEPEST+LITERAL; chunk-pipelined NCCL gather",
        "instances_total": total, "instances_per_rank_max": max(L.per), "chunks": L.n_chunks, "n_gpus": world,
        "ms_per_pass": ms_all, "schedules_per_s": 2 * total / (ms_all / 1000.0),
        "schedules_per_s_per_gpu": 2 * total / world / (ms_all / 1000.0),
        "ms_compute_only": ms_comp, "ms_gather_only": ms_gather,
        "gather_bytes_into_root": 2 * rec * (world - 1), "record_bytes_per_instance": 16 + 5 * V,
        "decisions_sha256": digest, "reps": args.c5_reps}}
    del T, bufs, roots, chunks
    torch.cuda.empty_cache()
    return res


class ChunkOut:
    """Outputs of instances [b0, b1) and queries [q0, q1): views into the full buffers."""

    def __init__(self, O, b0, b1, q0, q1):
        self.grid, self.grid_cfg = O.grid[b0:b1], O.grid_cfg[b0:b1]
        self.lsum, self.lmean, self.lcfg = O.lsum[b0:b1], O.lmean[b0:b1], O.lcfg[b0:b1]
        self.dec = [{k: d[k][b0:b1] for k in ("alloc", "cfg", "sum", "mean", "steps")} for d in O.dec]
        self.est = [e[q0:q1] for e in O.est]
        self.n = [n[q0:q1] for n in O.n]


def run_e2e(ek, h, w, T, rows, P, O, args, world):
    """Same step through the public API with HOST buffers: every step copies its inputs
    from pinned host memory and reads the decisions / estimates / objectives back.  The
    batch is split into chunks pipelined over three CUDA streams (host->device copy of
    chunk c+1 and device->host copy of chunk c-1 overlap the kernels of chunk c); the
    timed region spans all of it, copies included."""
    # host memory: every rank on this host pins its inputs and results; with several ranks
    # per host the e2e batch is the largest prefix of the step's batch that keeps all ranks'
    # pinned buffers within 60 % of the host's RAM (reported as batch_fraction)
    per_inst = sum(v[:1].numel() * v.element_size() for v in T.values()) + rows[:1].numel() * 2
    per_inst += sum(x[:1].numel() * x.element_size() for x in (O.grid, O.grid_cfg, O.lsum, O.lmean, O.lcfg))
    per_inst += sum(d[k][:1].numel() * d[k].element_size() for d in O.dec for k in ("sum", "mean", "steps", "alloc", "cfg"))
    per_q = sum(v[:1].numel() * v.element_size() for v in P.values())
    per_q += sum(x[:1].numel() * x.element_size() for x in O.est + O.n)
    need = w.B * per_inst + w.Q * per_q
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        ram = need * local_world * 2
    frac = min(1.0, 0.6 * ram / max(1, need * local_world))
    Be, Qe = max(1, int(w.B * frac)), max(1, int(w.Q * frac))
    w_full = w
    w = Workload(Be, w.N, Qe)
    T = {k: v[:Be] for k, v in T.items()}
    rows = rows[:Be]
    P = {k: v[:Qe] for k, v in P.items()}
    O = ChunkOut(O, 0, Be, 0, Qe)
    C = max(1, min(args.e2e_chunks, w.B, w.Q))
    bnd = [(w.B * c // C, w.B * (c + 1) // C, w.Q * c // C, w.Q * (c + 1) // C) for c in range(C)]
    host_T = {k: v.cpu().pin_memory() for k, v in T.items()}
    host_rows = rows.cpu().pin_memory()
    host_P = {k: v.cpu().pin_memory() for k, v in P.items()}

    def outs_of(o):   # every array read back: per-instance ones, per-query ones
        arr = [o.dec[0][k] for k in ("sum", "mean", "steps", "alloc", "cfg")]
        arr += [o.dec[1][k] for k in ("sum", "mean", "steps", "alloc", "cfg")]
        arr += [o.lsum, o.lmean, o.lcfg, o.grid, o.grid_cfg]
        q = [o.est[0], o.n[0], o.est[1], o.n[1]]
        return arr, q

    full_b, full_q = outs_of(O)
    host_b = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in full_b]
    host_q = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in full_q]
    h2d = sum(v.numel() * v.element_size() for v in list(host_T.values()) + [host_rows] + list(host_P.values()))
    d2h = sum(x.numel() * x.element_size() for x in full_b + full_q)
    s_in, s_comp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()
    comp_done = [None] * C
    out_done = [None] * C

    def e2e_step():
        in_ready = []
        for c, (b0, b1, q0, q1) in enumerate(bnd):
            with torch.cuda.stream(s_in):
                if comp_done[c] is not None:       # the previous step's kernels of chunk c read these
                    s_in.wait_event(comp_done[c])
                for k in T:
                    T[k][b0:b1].copy_(host_T[k][b0:b1], non_blocking=True)
                rows[b0:b1].copy_(host_rows[b0:b1], non_blocking=True)
                for k in P:
                    P[k][q0:q1].copy_(host_P[k][q0:q1], non_blocking=True)
                e = ev()
                e.record(s_in)
                in_ready.append(e)
        for c, (b0, b1, q0, q1) in enumerate(bnd):
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(in_ready[c])
                if out_done[c] is not None:        # the previous step's read-back of chunk c
                    s_comp.wait_event(out_done[c])
                wc = Workload(b1 - b0, w.N, q1 - q0)
                run_step(ek, h, wc, {k: v[b0:b1] for k, v in T.items()}, rows[b0:b1],
                         {k: v[q0:q1] for k, v in P.items()}, ChunkOut(O, b0, b1, q0, q1))
                e = ev()
                e.record(s_comp)
                comp_done[c] = e
            with torch.cuda.stream(s_out):
                s_out.wait_event(comp_done[c])
                for x, hx in zip(full_b, host_b):
                    hx[b0:b1].copy_(x[b0:b1], non_blocking=True)
                for x, hx in zip(full_q, host_q):
                    hx[q0:q1].copy_(x[q0:q1], non_blocking=True)
                e = ev()
                e.record(s_out)
                out_done[c] = e

    e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    t0.record(cur)
    for st in (s_in, s_comp, s_out):
        st.wait_event(t0)
    for _ in range(args.e2e_steps):
        e2e_step()
    for st in (s_in, s_comp, s_out):
        cur.wait_stream(st)
    t1.record(cur)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=rows.device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    return {"value": w.allocations() * world * args.e2e_steps / (ms / 1000.0), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms / args.e2e_steps, "steps": args.e2e_steps, "chunks": C,
            "batch_fraction": Be / w_full.B, "instances_per_rank": Be, "queries_per_rank": Qe,
            "read_back": "every counted unit's result: GRID values + configs of every cell, LIST sum/mean/configs "
                         "of every row, thief decisions (both modes), profile estimates + counts (both modes)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-inst", type=int, default=synth.CONFIG4.n_inst)
    ap.add_argument("--n-alloc", type=int, default=synth.CONFIG4.n_alloc)
    ap.add_argument("--n-query", type=int, default=synth.CONFIG3.n_query)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunks", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--no-context", dest="context", action="store_false")
    ap.add_argument("--context-v100", type=int, default=16384)
    ap.add_argument("--c5-inst", type=int, default=synth.CONFIG5.n_inst, help="config-5 instances in total (0: skip)")
    ap.add_argument("--c5-chunks", type=int, default=8)
    ap.add_argument("--c5-reps", type=int, default=2)
    ap.add_argument("--ref-inst", type=int, default=0, help="oracle sample instances (0: 256 per host thread)")
    ap.add_argument("--ref-query", type=int, default=0, help="oracle sample queries (0: 128 per host thread)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torch.distributed.run (the
        # driver's own N > 1 launch sets WORLD_SIZE and skips this)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    _stdout_to_stderr()   # after the re-launch: the ranks inherit the real stdout
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: launch one process per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # (NCCL's own log lines: run with NCCL_DEBUG=INFO NCCL_DEBUG_FILE=<file>; NCCL prints its
    # version banner on stdout at INFO, so the default run leaves NCCL_DEBUG unset and reports
    # the communicator's rank count from ncclCommCount in the JSON line instead)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
