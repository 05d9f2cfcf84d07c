"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the CPU oracle on
the same seeded inputs.

Bar (BASELINE.json north star): integer units, configs and exact Q32 objective
sums bit-exact; fp32 outputs (values, means, estimates) bit-exact as well,
because both sides follow the same one-rounding-per-operation contract
 -- strictly tighter than the north star's 1e-5 relative.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2012_10557_b200 import build
    build.build()
    from paper_2012_10557_b200 import ekya
    return ekya.Handle(0)


def ek():
    from paper_2012_10557_b200 import ekya
    return ekya


@pytest.fixture(scope="module")
def _dirty_inputs(h):
    pc = synth.ProfileConfig("p", 1184, 500, 27, 18)
    P = {k: v.cuda() for k, v in synth.profile_inputs(pc).items()}
    P["hist"].fill_(7.0)
    return P


@pytest.fixture(autouse=True)
def dirty_shared_memory(h, _dirty_inputs):
    """Before every test, leave out-of-range bit patterns (7.0) in every SM's shared memory:
    the profiler kernels stage a 54 KB history tile per query (invalid data: flagged, and
    cleared here), so a kernel that reads shared memory it never wrote fails parity instead
    of reading the zeros of a fresh context."""
    P = _dirty_inputs
    for mode in (ek().PROFILE_CLUSTER, ek().PROFILE_RADIUS):
        ek().profile_estimate(h, P["cur"], P["hist"], P["hist_acc"], P["fallback"], mode=mode)
    torch.cuda.synchronize()
    h.last_error()


def tables(cfg, lo=0, hi=None):
    T = synth.sched_tables(cfg, lo, hi)
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            cfg.units, cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)
    return {k: v.cuda() for k, v in T.items()}, inst


def args(cfg):
    return (cfg.units, cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)


def variant(cfg, **kw):
    return synth.SchedConfig(**{**cfg.__dict__, **kw})


SCHED_CASES = [
    ("c1", variant(synth.CONFIG1, n_inst=300)),
    ("c2", variant(synth.CONFIG2, n_inst=48)),
    ("c2-ragged", variant(synth.CONFIG2, n_inst=48, ragged=True)),
    ("c2-steal3", variant(synth.CONFIG2, n_inst=16, steal_units=3)),
    ("v1", variant(synth.CONFIG2, n_inst=16, n_streams=1, units=8)),
    ("nogamma", variant(synth.CONFIG2, n_inst=16, n_gamma=0)),
    ("u1", variant(synth.CONFIG1, n_inst=32, units=1)),
    ("odd", variant(synth.CONFIG2, n_inst=37, n_streams=7, n_gamma=31, n_lambda=5, units=53, a_min=0.0)),
    # > 4 instances per CTA: every mbarrier phase of LIST's two input buffers
    ("c1-many", variant(synth.CONFIG1, n_inst=1200)),
    # V x (U+1) too large for two LIST table sets in shared memory: the single-set path
    ("wide", variant(synth.CONFIG2, n_inst=20, n_streams=20, units=120)),
    # GRID beyond the staged position table (row located arithmetically), fewer warps per CTA
    ("bigU", variant(synth.CONFIG2, n_inst=6, n_streams=3, units=800)),
]


_SIGNED = {torch.uint16: torch.int16, torch.uint32: torch.int32, torch.uint64: torch.int64}


def pick(t, idx):
    """t[idx] for any dtype (unsigned types are indexed through a signed view)."""
    if t.dtype in _SIGNED:
        return t.view(_SIGNED[t.dtype])[idx].view(t.dtype)
    return t[idx]


def assert_eq(a, b, what):
    a = a.cpu().numpy() if torch.is_tensor(a) else a
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(a, b):
        bad = np.argwhere(a != b)
        raise AssertionError(f"{what}: {len(bad)} mismatches, first at {bad[:5].tolist()}: "
                             f"{a[tuple(bad[0])]} vs {b[tuple(bad[0])]}")


@pytest.mark.parametrize("name,cfg", SCHED_CASES, ids=[c[0] for c in SCHED_CASES])
def test_grid_bitexact(h, name, cfg):
    Td, inst = tables(cfg)
    grid, gcfg = ek().eval_grid(h, Td, *args(cfg))
    og, ocfg, bad = oracle.eval_grid(inst)
    assert bad == 0 and h.last_error() == 0
    assert_eq(grid, og, "grid values")
    assert_eq(gcfg, ocfg, "grid configs")


@pytest.mark.parametrize("name,cfg", SCHED_CASES, ids=[c[0] for c in SCHED_CASES])
def test_list_bitexact(h, name, cfg):
    Td, inst = tables(cfg)
    rows = synth.list_allocs(cfg, 300)
    s, mean, cfg_ = ek().eval_list(h, Td, rows.cuda(), *args(cfg))
    os_, om, ocf, bad = oracle.eval_list(inst, rows.numpy())
    assert bad == 0 and h.last_error() == 0
    assert_eq(s, os_, "sum_q32")
    assert_eq(mean, om, "mean")
    assert_eq(cfg_, ocf, "cfg")


def test_list_over_all_allocations_equals_bruteforce(h):
    """Eq. 1 on config 1: LIST over every allocation with sum <= U, argmax on the host,
    equals the oracle's brute force (value and lexicographically smallest allocation)."""
    import itertools
    cfg = variant(synth.CONFIG1, n_inst=64)
    Td, inst = tables(cfg)
    J, U = 4, cfg.units
    comps = np.array([c for c in itertools.product(range(U + 1), repeat=J) if sum(c) <= U], np.uint16)
    rows = torch.from_numpy(np.broadcast_to(comps, (cfg.n_inst,) + comps.shape).copy())
    s, mean, _ = ek().eval_list(h, Td, rows.cuda(), *args(cfg))
    s = s.cpu().numpy()
    ba, bc, bs, _ = oracle.bruteforce(inst)
    for b in range(cfg.n_inst):
        best = s[b].max()
        assert best == bs[b]
        first = np.flatnonzero(s[b] == best)[0]      # comps are in lexicographic order
        assert list(comps[first]) == list(ba[b])


def test_list_invalid_rows_and_data_errors(h):
    cfg = variant(synth.CONFIG2, n_inst=4)
    T = synth.sched_tables(cfg)
    T["cost"][3, 2, 5] = float("nan")                 # instance 3 invalid
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    Td = {k: v.cuda() for k, v in T.items()}
    rows = synth.list_allocs(cfg, 40)
    rows[0, 3, 4] = cfg.units + 1                      # entry > U
    rows[1, 7, 0] = int(rows[1, 7, 0]) + 3             # sum > U
    rows[2, 11, 19] = 65535                            # largest u16 entry (no out-of-table read)
    rows[2, 12, 0] = cfg.units                         # one stream takes every unit: valid
    rows[2, 12, 1:] = 0
    s, mean, c = ek().eval_list(h, Td, rows.cuda(), *args(cfg))
    assert h.last_error() == -6
    os_, om, ocf, bad = oracle.eval_list(inst, rows.numpy())
    assert bad == 3 + 40
    assert_eq(s, os_, "sum_q32")
    assert_eq(mean, om, "mean")
    assert_eq(c, ocf, "cfg")
    s, mean, c = ek().eval_list(h, Td, rows.cuda(), *args(cfg))
    assert h.last_error() == -6                        # EKYA_ERR_DATA, then cleared
    assert h.last_error() == 0


@pytest.mark.parametrize("mode", [0, 1], ids=["steepest", "literal"])
@pytest.mark.parametrize("name,cfg", SCHED_CASES, ids=[c[0] for c in SCHED_CASES])
def test_thief_bitexact(h, name, cfg, mode):
    Td, inst = tables(cfg)
    a, c, s, m, st = ek().thief_schedule(h, Td, *args(cfg), mode=mode)
    oa, oc, osum, omean, osteps, bad = oracle.thief(inst, mode)
    assert bad == 0 and h.last_error() == 0
    assert_eq(a, oa, "alloc")
    assert_eq(s, osum, "sum_q32")
    assert_eq(m, omean, "mean")
    assert_eq(c, oc, "cfg")
    assert_eq(st, osteps, "steps")
    assert (a.cpu().numpy().astype(np.int64).sum(1) == cfg.units).all()


def test_thief_invalid_instance_zeroed(h):
    cfg = variant(synth.CONFIG2, n_inst=6)
    T = synth.sched_tables(cfg)
    T["stale"][2, 1] = 1.5
    T["lam_factor"][4, 0, 0] = -0.1
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    Td = {k: v.cuda() for k, v in T.items()}
    a, c, s, m, st = ek().thief_schedule(h, Td, *args(cfg))
    oa, oc, osum, omean, osteps, bad = oracle.thief(inst, 0)
    assert bad == 2 and h.last_error() == -6
    assert_eq(a, oa, "alloc")
    assert_eq(s, osum, "sum")


def test_thief_persistent_claims_back_to_back(h):
    """LITERAL (and V > 16) run persistent warps claiming instances from a counter in the
    handle's device state that the last warp resets: launches of different sizes back to back,
    one with invalid instances (early exit inside the claim loop) and one empty, must each
    match the oracle -- a counter left non-zero would skip instances of the next launch."""
    base = variant(synth.CONFIG2, n_inst=5000, seed=77)
    T = synth.sched_tables(base)
    T["stale"][3, 0] = 1.5
    T["cost"][4998, 2, 1] = -1.0
    Td = {k: v.cuda() for k, v in T.items()}
    full = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(base))
    # instances are independent: one oracle run per mode serves every prefix (STEEPEST, one
    # instance per warp at V = 10, on the short prefixes only: its oracle is the slow one)
    ref = {1: oracle.thief(full, 1), 0: oracle.thief(full.subset(list(range(37))), 0)}
    for n in (5000, 1, 0, 37, 4737, 5000):   # > 4,736 resident warps: some claim twice
        Tn = {k: v[:n].contiguous() for k, v in Td.items()}
        for mode in ((1, 0) if n <= 37 else (1,)):
            a, c, s, m, st = ek().thief_schedule(h, Tn, *args(base), mode=mode)
            if n == 0:
                assert a.numel() == 0
                continue
            oa, oc, osum, omean, osteps, _ = ref[mode]
            bad = (n > 3) + (n > 4998)
            assert h.last_error() == (-6 if bad else 0)
            assert_eq(a, oa[:n], f"alloc n={n} mode={mode}")
            assert_eq(s, osum[:n], f"sum n={n} mode={mode}")
            assert_eq(c, oc[:n], f"cfg n={n} mode={mode}")
            assert_eq(st, osteps[:n], f"steps n={n} mode={mode}")


def test_thief_scaleout_shape(h):
    """Config 5 shape (V=100, U=800): LITERAL on 3 instances, STEEPEST on 1."""
    cfg = variant(synth.CONFIG5, n_inst=3)
    Td, inst = tables(cfg)
    a, c, s, m, st = ek().thief_schedule(h, Td, *args(cfg), mode=1)
    oa, oc, osum, omean, osteps, _ = oracle.thief(inst, 1)
    assert_eq(a, oa, "literal alloc")
    assert_eq(s, osum, "literal sum")
    assert_eq(c, oc, "literal cfg")
    Td1 = {k: v[:1].contiguous() for k, v in Td.items()}
    a, c, s, m, st = ek().thief_schedule(h, Td1, *args(cfg), mode=0)
    oa, oc, osum, omean, osteps, _ = oracle.thief(inst.subset([0]), 0)
    assert_eq(a, oa, "steepest alloc")
    assert_eq(s, osum, "steepest sum")
    assert_eq(st, osteps, "steepest steps")


def test_empty_batch(h):
    cfg = variant(synth.CONFIG2, n_inst=0)
    Td = {k: v.cuda() for k, v in synth.sched_tables(cfg).items()}
    a, c, s, m, st = ek().thief_schedule(h, Td, *args(cfg))
    assert a.shape == (0, 20)
    grid, _ = ek().eval_grid(h, Td, *args(cfg))
    assert grid.numel() == 0


def test_limits_rejected_synchronously(h):
    cfg = variant(synth.CONFIG2, n_inst=2)
    Td, _ = tables(cfg)
    e = ek()
    with pytest.raises(e.EkyaError) as ex:
        e.thief_schedule(h, Td, 65535, 1, 20.0, 0.4)
    assert ex.value.code == -2
    with pytest.raises(e.EkyaError):
        e.thief_schedule(h, Td, 80, 0, 20.0, 0.4)


# ---------------------------------------------------------------------------
# profiler
# ---------------------------------------------------------------------------
PROF_CASES = [
    ("dense", synth.ProfileConfig("p", 96, 500, 27, 18)),
    ("sparse", synth.ProfileConfig("p", 96, 500, 27, 18, sparse=True)),
    ("ragged", synth.ProfileConfig("p", 33, 137, 5, 3)),
    ("nohist", synth.ProfileConfig("p", 8, 0, 27, 18)),
    ("big-h", synth.ProfileConfig("p", 6, 1500, 27, 18)),
]


@pytest.mark.parametrize("mode", [0, 1], ids=["radius", "cluster"])
@pytest.mark.parametrize("name,pc", PROF_CASES, ids=[c[0] for c in PROF_CASES])
def test_profile_bitexact(h, name, pc, mode):
    P = synth.profile_inputs(pc)
    Pd = {k: v.cuda() for k, v in P.items()}
    est, n, cl = ek().profile_estimate(h, Pd["cur"], Pd["hist"], Pd["hist_acc"], Pd["fallback"], mode=mode,
                                       with_cluster=True)
    oe, on, ocl, bad, passes = oracle.profile(P["cur"].numpy(), P["hist"].numpy(), P["hist_acc"].numpy(),
                                              P["fallback"].numpy(), mode=mode, with_passes=True)
    assert bad == 0 and h.last_error() == 0
    assert_eq(n, on, "n_similar")
    assert_eq(est, oe, "estimate")
    if mode == 1:
        assert_eq(cl, ocl, "clusters")
        # the device's Lloyd pass counter (ekya_counters, used by bench.py's CLUSTER roofline)
        # equals the oracle's passes over the same queries
        c0 = h.counters()["lloyd_passes"]
        ek().profile_estimate(h, Pd["cur"], Pd["hist"], Pd["hist_acc"], Pd["fallback"], mode=mode)
        assert h.counters()["lloyd_passes"] - c0 == int(passes.sum())


BOTH_CASES = PROF_CASES + [
    ("h512", synth.ProfileConfig("p", 24, 512, 27, 18)),          # fused: the largest tile
    ("h513", synth.ProfileConfig("p", 12, 513, 27, 18)),          # not fused: two kernels
    ("h3", synth.ProfileConfig("p", 10, 3, 27, 18)),
    ("sparse-g1", synth.ProfileConfig("p", 40, 300, 27, 1, sparse=True)),
    ("h511", synth.ProfileConfig("p", 24, 511, 27, 18)),          # fused: the query in slot 511
    ("h255", synth.ProfileConfig("p", 24, 255, 27, 18)),          # fused: the query in slot 255
]


@pytest.mark.parametrize("name,pc", BOTH_CASES, ids=[c[0] for c in BOTH_CASES])
def test_profile_both_bitexact(h, name, pc):
    """ekya_profile_estimate_both: RADIUS and CLUSTER of the same queries (one history pass for
    k = 5, C = 27, H <= 512) equal the oracle's two modes element by element."""
    P = synth.profile_inputs(pc)
    Pd = {k: v.cuda() for k, v in P.items()}
    c0 = h.counters()["lloyd_passes"]
    er, nr, ec, nc, cl = ek().profile_estimate_both(h, Pd["cur"], Pd["hist"], Pd["hist_acc"], Pd["fallback"],
                                                    with_cluster=True)
    assert h.last_error() == 0
    args_ = tuple(P[k].numpy() for k in ("cur", "hist", "hist_acc", "fallback"))
    oe, on, _, bad = oracle.profile(*args_, mode=0)
    assert bad == 0
    assert_eq(nr, on, "n radius")
    assert_eq(er, oe, "estimate radius")
    oe, on, ocl, bad, passes = oracle.profile(*args_, mode=1, with_passes=True)
    assert_eq(nc, on, "n cluster")
    assert_eq(ec, oe, "estimate cluster")
    assert_eq(cl, ocl, "clusters")
    if pc.n_hist > 0:
        assert h.counters()["lloyd_passes"] - c0 == int(passes.sum())


def test_profile_both_invalid_queries(h):
    pc = synth.ProfileConfig("p", 5, 50, 27, 18)
    P = synth.profile_inputs(pc)
    P["hist"][2, 7, 3] = -0.5
    P["hist_acc"][4, 1, 1] = 2.0
    P["hist"][1, 49, 26] = float("nan")
    P["cur"][0, 5] = 1.5
    Pd = {k: v.cuda() for k, v in P.items()}
    er, nr, ec, nc, _ = ek().profile_estimate_both(h, Pd["cur"], Pd["hist"], Pd["hist_acc"], Pd["fallback"])
    assert h.last_error() == -6
    args_ = tuple(P[k].numpy() for k in ("cur", "hist", "hist_acc", "fallback"))
    for mode, (e, n) in enumerate(((er, nr), (ec, nc))):
        oe, on, _, bad = oracle.profile(*args_, mode=mode)
        assert bad == 4
        assert_eq(e, oe, f"estimate mode {mode}")
        assert_eq(n, on, f"n mode {mode}")


CLUSTER_EDGE = [
    # (name, config, k, max_iter): window counts at the 2-windows-per-thread boundaries of the
    # multi-query CLUSTER kernel, k at its register-cache limits, capped iteration counts
    ("h256-k8", synth.ProfileConfig("p", 40, 256, 27, 18), 8, 100),
    ("h257-k1", synth.ProfileConfig("p", 40, 257, 27, 18), 1, 100),
    ("h512-k5", synth.ProfileConfig("p", 24, 512, 27, 18), 5, 100),
    ("h513-k5", synth.ProfileConfig("p", 12, 513, 27, 18), 5, 100),
    ("h500-k5-iter0", synth.ProfileConfig("p", 30, 500, 27, 18), 5, 0),
    ("h500-k5-iter1", synth.ProfileConfig("p", 30, 500, 27, 18), 5, 1),
    ("h500-k7-iter3", synth.ProfileConfig("p", 30, 500, 27, 18), 7, 3),
    ("c32-g1", synth.ProfileConfig("p", 20, 300, 32, 1), 5, 100),
    ("c1-g40", synth.ProfileConfig("p", 20, 90, 1, 40), 3, 100),
    ("k9-fallback", synth.ProfileConfig("p", 10, 500, 27, 18), 9, 100),
    ("h3-k5", synth.ProfileConfig("p", 10, 3, 27, 18), 5, 100),
    # the query's window slot (first unused slot, H < 512) at its extremes: slot 511 (last
    # thread's second window) and slot 255 (last thread's first window); C = 26 puts the
    # count-carrying lane C next to a real column lane
    ("h511-k5", synth.ProfileConfig("p", 24, 511, 27, 18), 5, 100),
    ("h255-k5", synth.ProfileConfig("p", 24, 255, 27, 18), 5, 100),
    ("c26-h400", synth.ProfileConfig("p", 24, 400, 26, 18), 5, 100),
]


@pytest.mark.parametrize("name,pc,k,it", CLUSTER_EDGE, ids=[c[0] for c in CLUSTER_EDGE])
def test_cluster_edges_bitexact(h, name, pc, k, it):
    P = synth.profile_inputs(pc)
    Pd = {kk: v.cuda() for kk, v in P.items()}
    est, n, cl = ek().profile_estimate(h, Pd["cur"], Pd["hist"], Pd["hist_acc"], Pd["fallback"], mode=1, k=k,
                                       max_iter=it, with_cluster=True)
    oe, on, ocl, bad = oracle.profile(P["cur"].numpy(), P["hist"].numpy(), P["hist_acc"].numpy(),
                                      P["fallback"].numpy(), mode=1, k=k, max_iter=it)
    assert bad == 0 and h.last_error() == 0
    assert_eq(cl, ocl, "clusters")
    assert_eq(n, on, "n_similar")
    assert_eq(est, oe, "estimate")


def test_profile_invalid_query(h):
    pc = synth.ProfileConfig("p", 5, 50, 27, 18)
    P = synth.profile_inputs(pc)
    P["hist"][2, 7, 3] = -0.5
    P["hist_acc"][4, 1, 1] = 2.0
    P["hist"][1, 49, 26] = float("nan")       # last class of the last window
    P["hist"][3, 0, 0] = float("inf")
    Pd = {k: v.cuda() for k, v in P.items()}
    for mode in (0, 1):
        est, n, _ = ek().profile_estimate(h, Pd["cur"], Pd["hist"], Pd["hist_acc"], Pd["fallback"], mode=mode)
        oe, on, _, bad = oracle.profile(*(P[k].numpy() for k in ("cur", "hist", "hist_acc", "fallback")),
                                        mode=mode)
        assert bad == 4 and h.last_error() == -6
        assert_eq(est, oe, "estimate")
        assert_eq(n, on, "n")


def test_profile_output_feeds_thief_tables(h):
    """With q = b*V + v, out_est is the post table of a batch (ABI contract)."""
    cfg = variant(synth.CONFIG2, n_inst=8)
    Td, inst = tables(cfg)
    pc = synth.ProfileConfig("p", cfg.n_inst * cfg.n_streams, 200, 27, cfg.n_gamma)
    P = {k: v.cuda() for k, v in synth.profile_inputs(pc).items()}
    est, n, _ = ek().profile_estimate(h, P["cur"], P["hist"], P["hist_acc"], P["fallback"])
    Td["post"] = est.view(cfg.n_inst, cfg.n_streams, cfg.n_gamma).contiguous()
    a, c, s, m, st = ek().thief_schedule(h, Td, *args(cfg))
    inst2 = oracle.Instances(inst.stale, inst.cost, Td["post"].cpu().numpy(), inst.lam_min_units,
                             inst.lam_factor, *args(cfg))
    oa, oc, osum, *_ = oracle.thief(inst2, 0)
    assert_eq(a, oa, "alloc")
    assert_eq(s, osum, "sum")


# ---------------------------------------------------------------------------
# full BASELINE sizes, in the launch configuration bench.py times, sampled
# ---------------------------------------------------------------------------
def test_config4_full_batch_sampled(h):
    cfg = synth.CONFIG4
    Td = synth.sched_tables(cfg, device="cuda")
    e = ek()
    a, c, s, m, st = e.thief_schedule(h, Td, *args(cfg), mode=0)
    grid, gcfg = e.eval_grid(h, Td, *args(cfg))
    rows = synth.list_allocs(cfg, 256, 0, cfg.n_inst, device="cuda")
    ls, lm, lc = e.eval_list(h, Td, rows, *args(cfg))
    assert h.last_error() == 0
    assert (a.cpu().numpy().astype(np.int64).sum(1) == cfg.units).all()
    sample = [0, 1, 4095, 31337, 65535] + list(np.random.default_rng(7).integers(0, cfg.n_inst, 11))
    Tc = synth.sched_tables(cfg)              # CPU generation of the same instances
    for k in Tc:
        assert torch.equal(pick(Tc[k], sample), pick(Td[k], sample).cpu()), f"device/host generator mismatch: {k}"
    inst = oracle.Instances(*(pick(Tc[k], sample).numpy() for k in ("stale", "cost", "post", "lam_min_units",
                                                              "lam_factor")), *args(cfg))
    oa, oc, osum, omean, osteps, _ = oracle.thief(inst, 0)
    assert_eq(pick(a, sample), oa, "alloc")
    assert_eq(pick(s, sample), osum, "sum")
    assert_eq(pick(c, sample), oc, "cfg")
    assert_eq(pick(m, sample), omean, "mean")
    assert_eq(pick(st, sample), osteps, "steps")
    # LITERAL over the same full batch
    a, c, s, m, st = e.thief_schedule(h, Td, *args(cfg), mode=1)
    assert h.last_error() == 0
    oa, oc, osum, omean, osteps, _ = oracle.thief(inst, 1)
    assert_eq(pick(a, sample), oa, "literal alloc")
    assert_eq(pick(s, sample), osum, "literal sum")
    assert_eq(pick(c, sample), oc, "literal cfg")
    assert_eq(pick(m, sample), omean, "literal mean")
    assert_eq(pick(st, sample), osteps, "literal steps")
    og, ocfg, _ = oracle.eval_grid(inst)
    assert_eq(pick(grid, sample), og, "grid")
    assert_eq(pick(gcfg, sample), ocfg, "grid cfg")
    os_, om, ocf, _ = oracle.eval_list(inst, pick(rows, sample).cpu().numpy())
    assert_eq(pick(ls, sample), os_, "list sum")
    assert_eq(pick(lm, sample), om, "list mean")
    assert_eq(pick(lc, sample), ocf, "list cfg")


def test_config4_list_bench_launch_sampled(h):
    """LIST in exactly the launch configuration bench.py times: 65,536 config-4 instances x
    4,096 rows, generated on the device by bench.gen_list_rows, evaluated by the same
    ekya_eval_allocations call as bench.run_step with all three outputs (sum, mean, cfg).
    At 4,096 rows the kernel builds stream tables as one task per stream, double-buffered
    across the ~443 instances of each CTA, so builds of instance j+1 overlap rows of j.
    24 sampled instances (all 4,096 rows each, incl. both ends of the batch) vs the oracle."""
    import bench
    e = ek()
    dev = torch.device("cuda")
    w = bench.Workload(synth.CONFIG4.n_inst, synth.CONFIG4.n_alloc, 0)
    Td = synth.sched_tables(w.cfg, 0, w.B, device=dev)
    rows = bench.gen_list_rows(w, dev)
    ls = torch.empty((w.B, w.N), dtype=torch.uint64, device=dev)
    lm = torch.empty((w.B, w.N), dtype=torch.float32, device=dev)
    lc = torch.empty((w.B, w.N, w.V), dtype=torch.uint8, device=dev)
    e.ekya_eval_allocations(h, e.dims_from(Td, *w.args), e.make_tables(**Td), e.EVAL_LIST, w.N, rows, ls, lm, lc)
    torch.cuda.synchronize()
    assert h.last_error() == 0
    rng = np.random.default_rng(11)
    sample = [0, 1, 442, 443, 444, 32767, 65534, 65535] + list(rng.integers(0, w.B, 16))
    Tc = synth.sched_tables(w.cfg)            # CPU generation of the same instances
    inst = oracle.Instances(*(pick(Tc[k], sample).numpy() for k in ("stale", "cost", "post", "lam_min_units",
                                                              "lam_factor")), *w.args)
    rc = pick(rows, sample).cpu()
    for i, b in enumerate(sample):
        assert torch.equal(rc[i], synth.list_allocs(w.cfg, w.N, b, b + 1)[0]), "device/host row generator mismatch"
    os_, om, ocf, bad = oracle.per_instance_parallel(oracle.eval_list, inst, rc.numpy())
    assert bad == 0
    assert_eq(pick(ls, sample), os_, "list sum")
    assert_eq(pick(lm, sample), om, "list mean")
    assert_eq(pick(lc, sample), ocf, "list cfg")


def config5_device_tables(B, dev):
    """Config-5 tables (V = 100, U = 800) for instances [0, B) on the device, in chunks."""
    cfg = variant(synth.CONFIG5, n_inst=B)
    parts = [synth.sched_tables(cfg, b0, min(B, b0 + 16384), device=dev) for b0 in range(0, B, 16384)]
    return cfg, {k: torch.cat([p[k] for p in parts]) for k in parts[0]}


def test_config5_sample_both_modes(h):
    """Config 5 (V = 100, U = 800) thief in both modes on a 131,072-instance batch (the
    per-GPU shard size of the 1M-instance, 8-GPU run, rounded up), sampled at instances
    0..63 ("parity-check a fixed sample (instances 0...63)") against the oracle
    on a thread pool of all host cores (the oracle's STEEPEST costs ~1e2 core-s per
    config-5 instance)."""
    e = ek()
    cfg, Td = config5_device_tables(131072, torch.device("cuda"))
    sample = list(range(64))
    Tc = synth.sched_tables(cfg, 0, 64)
    inst = oracle.Instances(*(Tc[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    for mode in (1, 0):
        a, c, s, m, st = e.thief_schedule(h, Td, *args(cfg), mode=mode)
        assert h.last_error() == 0
        oa, oc, osum, omean, osteps, bad = oracle.per_instance_parallel(oracle.thief, inst, mode)
        assert bad == 0
        assert_eq(a[:64], oa, f"alloc mode {mode}")
        assert_eq(s[:64], osum, f"sum mode {mode}")
        assert_eq(c[:64], oc, f"cfg mode {mode}")
        assert_eq(m[:64], omean, f"mean mode {mode}")
        assert_eq(st[:64], osteps, f"steps mode {mode}")
        assert (a.to(torch.int64).sum(1) == cfg.units).all()


def test_gather_decisions_one_rank_both_paths(h):
    """The multi-GPU data plane on one GPU: thief decisions written by the kernels straight
    into shard.RecordLayout's chunked record views (device), gathered chunk by chunk with
    ekya_gather_decisions -- without a communicator (device copy) and through a one-rank NCCL
    communicator (ncclGather) -- unpacked at the root and compared with the oracle."""
    from paper_2012_10557_b200 import shard
    e = ek()
    cfg = variant(synth.CONFIG2, n_inst=301)
    Td, inst = tables(cfg)
    oa, oc, osum, omean, osteps, _ = oracle.thief(inst, 0)
    h1 = e.Handle(0)
    e.ekya_comm_init(h1, e.ekya_comm_unique_id(), 1, 0)
    assert e.ekya_comm_info(h1) == (1, 0) and e.ekya_comm_info(h) == (1, 0)
    for hh in (h, h1):
        L = shard.RecordLayout(cfg.n_inst, 1, cfg.n_streams, n_chunks=4)
        buf = torch.zeros(L.rank_bytes, dtype=torch.uint8, device="cuda")
        root = torch.zeros(L.root_bytes, dtype=torch.uint8, device="cuda")
        dims = e.dims_from(Td, *args(cfg))
        side = torch.cuda.Stream()
        for c in range(L.n_chunks):
            b0, b1 = L.chunk_range(0, c)
            v = L.views(buf, 0, c)
            Tc = {k: x[b0:b1] for k, x in Td.items()}
            dc = e.dims_from(Tc, *args(cfg))
            e.ekya_thief_schedule(hh, dc, e.make_tables(**Tc), 0, v["alloc"], v["cfg"], v["sum"], v["mean"],
                                  v["steps"])
            ev = torch.cuda.Event()
            ev.record()
            side.wait_event(ev)
            e.ekya_gather_decisions(hh, L.local_chunk(buf, c), L.root_chunk(root, c), root=0, stream=side)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        assert hh.last_error() == 0
        got = L.unpack(root)
        assert_eq(got["alloc"], oa, "gathered alloc")
        assert_eq(got["cfg"], oc, "gathered cfg")
        assert_eq(got["sum"], osum, "gathered sum")
        assert_eq(got["mean"], omean, "gathered mean")
        assert_eq(got["steps"], osteps, "gathered steps")
        assert torch.equal(root, buf)      # one rank: the root holds the rank's buffer byte for byte
    del dims
    h1.close()


def test_config3_fused_full_batch_sampled(h):
    """The bench's profile launch (both estimates in one pass) at config 3's full size,
    sampled against the oracle's two modes."""
    pc = synth.CONFIG3
    e = ek()
    P = synth.profile_inputs(pc, device="cuda")
    er, nr, ec, nc, cl = e.profile_estimate_both(h, P["cur"], P["hist"], P["hist_acc"], P["fallback"],
                                                 with_cluster=True)
    assert h.last_error() == 0
    del P
    sample = [0, 1, 65535] + list(np.random.default_rng(9).integers(0, pc.n_query, 9))
    for q in sample:
        Pc = synth.profile_inputs(pc, q, q + 1)
        a_ = tuple(Pc[k].numpy() for k in ("cur", "hist", "hist_acc", "fallback"))
        oe, on, _, _ = oracle.profile(*a_, mode=0)
        assert_eq(er[q:q + 1], oe, f"radius est q={q}")
        assert_eq(nr[q:q + 1], on, f"radius n q={q}")
        oe, on, ocl, _ = oracle.profile(*a_, mode=1)
        assert_eq(ec[q:q + 1], oe, f"cluster est q={q}")
        assert_eq(nc[q:q + 1], on, f"cluster n q={q}")
        assert_eq(cl[q:q + 1], ocl, f"cluster q={q}")


def test_config3_full_batch_sampled(h):
    pc = synth.CONFIG3
    e = ek()
    for mode in (0, 1):
        P = synth.profile_inputs(pc, device="cuda")
        est, n, cl = e.profile_estimate(h, P["cur"], P["hist"], P["hist_acc"], P["fallback"], mode=mode,
                                        with_cluster=(mode == 1))
        assert h.last_error() == 0
        sample = [0, 1, 65535] + list(np.random.default_rng(8).integers(0, pc.n_query, 9))
        del P
        for q in sample:
            Pc = synth.profile_inputs(pc, q, q + 1)
            oe, on, ocl, _ = oracle.profile(*(Pc[k].numpy() for k in ("cur", "hist", "hist_acc", "fallback")),
                                            mode=mode)
            assert_eq(est[q:q + 1], oe, f"est q={q}")
            assert_eq(n[q:q + 1], on, f"n q={q}")
            if mode == 1:
                assert_eq(cl[q:q + 1], ocl, f"cluster q={q}")


def test_next_rows_full_batch_sampled(h):
    """The NEXT rows at the bench's full sizes and launch configuration, on sampled outputs:
    the window timeline, uniform baseline, Pareto frontier and placement over config 4's
    65,536 instances; pruning over config 3's 65,536 histories with config-4 costs."""
    cfg = synth.CONFIG4
    Td = synth.sched_tables(cfg, device="cuda")
    e = ek()
    avg, ev, done = e.window_schedule(h, Td, *args(cfg))
    ua, uc, us, um = e.uniform_schedule(h, Td, *args(cfg))
    par = e.pareto(h, Td["cost"], Td["post"])
    a, *_ = e.thief_schedule(h, Td, *args(cfg))
    pj, pq, pg, npc, load = e.place(h, a, cfg.units, 8)
    assert h.last_error() == 0
    sample = [0, 65535] + list(np.random.default_rng(9).integers(0, cfg.n_inst, 6))
    Tc = {k: pick(v, sample).cpu() for k, v in Td.items()}
    inst = oracle.Instances(*(Tc[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    oavg, oev, odone, _ = oracle.window(inst)
    assert_eq(pick(ev, sample), oev, "window invocations")
    assert_eq(pick(done, sample), odone, "window completion times")
    assert_eq(pick(avg, sample), oavg, "window average")
    oa, oc, osum, _, _ = oracle.uniform(inst)
    assert_eq(pick(ua, sample), oa, "uniform alloc")
    assert_eq(pick(us, sample), osum, "uniform sum")
    assert_eq(pick(par, sample), oracle.pareto(inst.cost, inst.post), "pareto mask")
    opj, opq, opg, onp, oload, _ = oracle.place(pick(a, sample).cpu().numpy(), cfg.units, 8)
    assert_eq(pick(pj, sample), opj, "piece jobs")
    assert_eq(pick(pg, sample), opg, "piece gpus")
    assert_eq(pick(load, sample), oload, "gpu loads")
    # pruning: config-3 histories (device generation in chunks), config-4 costs of the first
    # 65,536 streams
    pc = synth.CONFIG3
    acc = torch.empty((pc.n_query, pc.n_hist, pc.n_gamma), device="cuda")
    for q0 in range(0, pc.n_query, 4096):
        acc[q0:q0 + 4096] = synth.profile_inputs(pc, q0, q0 + 4096, device="cuda")["hist_acc"]
    cost = Td["cost"].reshape(-1, Td["cost"].shape[-1])[:pc.n_query, :pc.n_gamma].contiguous()
    keep = e.prune_configs(h, cost, acc, 0.05)
    assert h.last_error() == 0
    qs = [0, 65535] + list(np.random.default_rng(10).integers(0, pc.n_query, 30))
    ok, bad = oracle.prune(pick(cost, qs).cpu().numpy(), pick(acc, qs).cpu().numpy(), 0.05)
    assert bad == 0
    assert_eq(pick(keep, qs), ok, "prune keep mask")


def adversarial_ties(n_inst=24):
    """Config-2 instances edited so the config choice hits every tie path: duplicated
    gamma (exact ties -> lowest index), 1-ulp neighbours (near ties inside 2^-21), a zero
    and a subnormal lambda factor (zero / subnormal products), post == stale (ties with the
    no-retraining choice)."""
    cfg = variant(synth.CONFIG2, n_inst=n_inst, a_min=0.0)   # a_MIN = 0 admits zero-accuracy lambdas
    T = synth.sched_tables(cfg)
    cost, post, stale, lf = T["cost"], T["post"], T["stale"], T["lam_factor"]
    cost[:, 0, 1:4] = cost[:, 0, 0:1]
    post[:, 0, 1:4] = post[:, 0, 0:1]
    p1 = post[:, 1, 0:1]
    post[:, 1, 1:2] = torch.nextafter(p1, torch.ones_like(p1))
    post[:, 1, 2:3] = torch.nextafter(p1, torch.zeros_like(p1))
    cost[:, 1, 1:3] = cost[:, 1, 0:1]
    lf[:, 2, :] = 0.0
    lf[:, 3, 1:] = 1e-39
    post[:, 4, :] = stale[:, 4:5]
    cost[:, 5, :] = cost[:, 5, 0:1]            # every gamma the same cost, posts differ
    return cfg, T


def test_ties_grid_list_thief_bitexact(h):
    cfg, T = adversarial_ties()
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    Td = {k: v.cuda() for k, v in T.items()}
    grid, gcfg = ek().eval_grid(h, Td, *args(cfg))
    og, ocfg, bad = oracle.eval_grid(inst)
    assert bad == 0 and h.last_error() == 0
    assert_eq(grid, og, "grid values")
    assert_eq(gcfg, ocfg, "grid configs")
    rows = synth.list_allocs(cfg, 4096)        # the many-rows LIST path (one build task per stream)
    s, mean, c = ek().eval_list(h, Td, rows.cuda(), *args(cfg))
    os_, om, ocf, _ = oracle.eval_list(inst, rows.numpy())
    assert_eq(s, os_, "list sum")
    assert_eq(c, ocf, "list cfg")
    for mode in (0, 1):
        a, cc, ts, tm, st = ek().thief_schedule(h, Td, *args(cfg), mode=mode)
        oa, oc, osum, omean, osteps, _ = oracle.thief(inst, mode)
        assert_eq(a, oa, f"thief alloc {mode}")
        assert_eq(cc, oc, f"thief cfg {mode}")
        assert_eq(ts, osum, f"thief sum {mode}")


# ---------------------------------------------------------------------------
# NEXT-4: placement onto GPUs and the checkpoint decision
# ---------------------------------------------------------------------------
def _place_cmp(h, alloc, units, gpus):
    pj, pq, pg, npc, load = ek().place(h, alloc.cuda(), units, gpus)
    opj, opq, opg, onpc, oload, bad = oracle.place(alloc.numpy(), units, gpus)
    assert_eq(npc, onpc, "n_pieces")
    assert_eq(pj, opj, "piece_job")
    assert_eq(pq, opq, "piece_q")
    assert_eq(pg, opg, "piece_gpu")
    assert_eq(load, oload, "gpu_load")
    return bad


@pytest.mark.parametrize("name,cfg,gpus", [("c2", variant(synth.CONFIG2, n_inst=256), 8),
                                           ("c5", variant(synth.CONFIG5, n_inst=48), 80)],
                         ids=["config2-8gpu", "config5-80gpu"])
def test_place_thief_decisions_bitexact(h, name, cfg, gpus):
    """The thief's decisions placed on the cluster's GPUs (delta = G/U GPU per unit)."""
    Td, _ = tables(cfg)
    a, *_ = ek().thief_schedule(h, Td, *args(cfg))
    assert _place_cmp(h, a.cpu(), cfg.units, gpus) == 0 and h.last_error() == 0


def test_place_random_edges_bitexact(h):
    rng = np.random.default_rng(21)
    for J, U, G in [(1, 1, 1), (3, 10, 2), (20, 80, 8), (7, 65534, 128), (64, 100, 100), (33, 7, 33),
                    (200, 800, 80), (5, 3, 96)]:
        B = 64
        w = rng.integers(0, 6, (B, J))
        a = np.floor(w / np.maximum(1, w.sum(1, keepdims=True)) * U).astype(np.int64)
        a[0] = 0
        a[1] = 0
        a[1, 0] = U                                    # one job takes everything
        if J > 1:
            a[2, :2] = U                               # sum > U: data error
        bad = _place_cmp(h, torch.from_numpy(a.astype(np.uint16)), U, G)
        assert bad == (1 if J > 1 else 0)
        assert h.last_error() == (-6 if bad else 0)


def test_checkpoint_bitexact(h):
    rng = np.random.default_rng(22)
    n = 100_000
    T = rng.uniform(10, 300, n).astype(np.float32)
    tau = (T * rng.uniform(0, 1, n)).astype(np.float32)
    t = (tau * rng.uniform(0, 1, n)).astype(np.float32)
    a, ast, A = (rng.uniform(0, 1, n).astype(np.float32) for _ in range(3))
    dl = rng.uniform(0, 20, n).astype(np.float32)
    t[:5] = tau[:5] + 1.0                              # invalid: t > tau
    A[5] = 1.5
    dl[6] = -1.0
    ast[7:100] = a[7:100]                              # no gain
    dl[100:200] = 0.0
    out = ek().checkpoint_decide(h, *(torch.from_numpy(x).cuda() for x in (tau, t, T, a, ast, A, dl)))
    oo, bad = oracle.checkpoint(tau, t, T, a, ast, A, dl)
    assert bad == 7 and h.last_error() == -6
    assert_eq(out, oo, "checkpoint")


def test_next_rows_exact_ties_and_clamp(h):
    """The oracle pins' boundary cases on the GPU: CK1's exact tie (no checkpoint) and its
    nextafter neighbour; U2's tied highest post (lowest index); CF2's all-zero-SSE grid
    (c = 0) and CF3's clamp at 0."""
    f = lambda *xs: [torch.tensor(x, dtype=torch.float32).cuda() for x in xs]
    up = float(np.nextafter(np.float32(0.625), np.float32(1)))
    args_ck = ([30, 30], [20, 20], [100, 100], [0.5, 0.5], [0.625, up], [0.5, 0.5], [2.5, 2.5])
    out = ek().checkpoint_decide(h, *f(*args_ck))
    oo, bad = oracle.checkpoint(*args_ck)
    assert bad == 0 and oo.tolist() == [0, 1]
    assert_eq(out, oo, "checkpoint tie")
    c = variant(synth.CONFIG2, n_inst=40)
    T = synth.sched_tables(c)
    T["post"] = T["post"] * 0.5
    for b in range(40):
        for v in range(T["post"].shape[1]):
            T["post"][b, v, (3 + b + v) % 18] = 1.0
            T["post"][b, v, (11 + 2 * b + v) % 18] = 1.0
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(c))
    a, cf, sm, m = ek().uniform_schedule(h, {k: v.cuda() for k, v in T.items()}, *args(c))
    oa, oc, osum, omean, bad = oracle.uniform(inst)
    assert bad == 0
    assert_eq(cf, oc, "uniform tied cfg")
    assert_eq(sm, osum, "uniform tied sum")
    acc = np.array([[0.5] * 5, [0.0, 1 / 64, 6 / 64, 6 / 64, 6 / 64], [0.0, 0.0, 3 / 64, 6 / 64, 6 / 64]],
                   np.float32)
    K = np.array([7, 1, 1], np.int32)
    pred, prm = ek().curve_fit(h, torch.from_numpy(acc).cuda(), torch.from_numpy(K).cuda())
    op, oprm, bad = oracle.curve_fit(acc, K)
    assert bad == 0
    assert_eq(pred, op, "curve fit pred")
    assert_eq(prm, oprm, "curve fit params")


# ---------------------------------------------------------------------------
# NEXT-3: uniform baseline and Pareto frontier
# ---------------------------------------------------------------------------
UNIFORM_CASES = [("c2-highest", variant(synth.CONFIG2, n_inst=96), -1, 0.5),
                 ("c2-ragged-g3-w07", variant(synth.CONFIG2, n_inst=64, ragged=True), 3, 0.7),
                 ("c2-none-w025", variant(synth.CONFIG2, n_inst=64), 0, 0.25),
                 ("c1-g2-w09", variant(synth.CONFIG1, n_inst=300), 2, 0.9),
                 ("odd-highest", variant(synth.CONFIG2, n_inst=37, n_streams=37, n_gamma=31, units=100), -1, 0.5),
                 ("nogamma", variant(synth.CONFIG2, n_inst=16, n_gamma=0), -1, 0.5)]


@pytest.mark.parametrize("name,cfg,g,w", UNIFORM_CASES, ids=[c[0] for c in UNIFORM_CASES])
def test_uniform_bitexact(h, name, cfg, g, w):
    Td, inst = tables(cfg)
    a, c, s, m = ek().uniform_schedule(h, Td, *args(cfg), fixed_gamma=g, inference_weight=w)
    oa, oc, osum, omean, bad = oracle.uniform(inst, g, w)
    assert bad == 0 and h.last_error() == 0
    assert_eq(a, oa, "alloc")
    assert_eq(c, oc, "cfg")
    assert_eq(s, osum, "sum")
    assert_eq(m, omean, "mean")


def test_uniform_invalid_instance_zeroed(h):
    cfg = variant(synth.CONFIG2, n_inst=6)
    T = synth.sched_tables(cfg)
    T["post"][2, 1, 3] = 1.5
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    a, c, s, m = ek().uniform_schedule(h, {k: v.cuda() for k, v in T.items()}, *args(cfg))
    oa, oc, osum, omean, bad = oracle.uniform(inst)
    assert bad == 1 and h.last_error() == -6
    assert_eq(a, oa, "alloc")
    assert_eq(s, osum, "sum")


def test_pareto_bitexact(h):
    cfg = variant(synth.CONFIG2, n_inst=512, ragged=True)
    Td, inst = tables(cfg)
    m = ek().pareto(h, Td["cost"], Td["post"])
    assert_eq(m, oracle.pareto(inst.cost, inst.post), "pareto mask (tables)")
    rng = np.random.default_rng(41)
    for n in (1, 2, 7, 31):
        c = (rng.choice([1.0, 2.0, 3.0, 5.0], (2000, n)) * rng.integers(1, 4, (2000, n))).astype(np.float32)
        p = np.round(rng.uniform(0, 1, (2000, n)), 1).astype(np.float32)
        c[rng.uniform(size=c.shape) < 0.1] = np.inf
        m = ek().pareto(h, torch.from_numpy(c).cuda(), torch.from_numpy(p).cuda())
        assert_eq(m, oracle.pareto(c, p), f"pareto mask n={n}")
    assert h.last_error() == 0
    # invalid data (R-ERR): NaN / negative / -inf costs, real accuracies outside [0, 1]
    c = (rng.choice([1.0, 2.0, 3.0], (3000, 18))).astype(np.float32)
    p = rng.uniform(0, 1, (3000, 18)).astype(np.float32)
    c[rng.uniform(size=c.shape) < 0.1] = np.inf
    p[np.isinf(c)] = 9.0                                  # padding accuracies are ignored
    c[5, 3], c[7, 0], c[9, 17] = np.nan, -1.0, -np.inf
    p[11, 2], p[13, 4] = 1.5, np.nan
    c[11, 2] = c[13, 4] = 1.0
    m = ek().pareto(h, torch.from_numpy(c).cuda(), torch.from_numpy(p).cuda())
    om, bad = oracle.pareto(c, p, with_bad=True)
    assert bad == 5 and h.last_error() == -6
    assert_eq(m, om, "pareto mask (invalid sets)")
    with pytest.raises(ek().EkyaError) as ex:
        ek().pareto(h, torch.zeros((4, 0), device="cuda"), torch.zeros((4, 0), device="cuda"))
    assert ex.value.code == -3


@pytest.mark.parametrize("name,pc", [c for c in PROF_CASES if c[0] != "big-h"], ids=[c[0] for c in PROF_CASES
                                                                                    if c[0] != "big-h"])
def test_prune_profile_histories_bitexact(h, name, pc):
    """History-based pruning (PN1-PN3) on the profiler's history accuracies (dense, sparse,
    ragged, no history) with the schedulers' cost tables, at three margins."""
    P = synth.profile_inputs(pc)
    acc = P["hist_acc"].numpy()
    Q, G = acc.shape[0], acc.shape[2]
    cfg = variant(synth.CONFIG2, n_inst=(Q + 9) // 10, ragged=True)
    _, inst = tables(cfg)
    cost = np.ascontiguousarray(inst.cost.reshape(-1, inst.cost.shape[-1])[:Q, :G])
    for m in (0.0, 0.02, 0.1):
        keep = ek().prune_configs(h, torch.from_numpy(cost).cuda(), torch.from_numpy(acc).cuda(), m)
        ok, bad = oracle.prune(cost, acc, m)
        assert bad == 0 and h.last_error() == 0
        assert_eq(keep, ok, f"keep mask margin={m}")


def test_prune_random_edges_bitexact(h):
    """Tie-heavy costs and accuracies, unmeasured and padding configs, every register-bound
    instantiation (n <= 8, 18, 31), window counts around the 32-window staging, invalid
    streams."""
    rng = np.random.default_rng(43)
    for n, H in [(1, 1), (5, 0), (8, 31), (9, 32), (18, 33), (18, 500), (31, 65), (31, 7)]:
        Q = 300
        c = (rng.choice([1.0, 2.0, 3.0, 5.0], (Q, n)) * rng.integers(1, 3, (Q, n))).astype(np.float32)
        c[rng.uniform(size=c.shape) < 0.1] = np.inf
        A = np.round(rng.uniform(0, 1, (Q, H, n)), 1).astype(np.float32)
        A[rng.uniform(size=A.shape) < 0.2] = np.nan
        A[Q // 2:] = rng.uniform(0, 1, A[Q // 2:].shape).astype(np.float32)   # no ties
        if H:
            A[7, :, :] = np.nan                                                  # nothing measured
            A[9, 0, 0] = 1.5                                                     # invalid unless padding
        c[11, 0] = np.nan                                                        # invalid
        c[13, -1] = -1.0                                                         # invalid
        for m in (0.0, 0.15):
            keep = ek().prune_configs(h, torch.from_numpy(c).cuda(), torch.from_numpy(A).cuda(), m)
            ok, bad = oracle.prune(c, A, m)
            assert bad > 0 and h.last_error() == -6
            assert_eq(keep, ok, f"keep mask n={n} H={H} margin={m}")


def test_prune_equal_costs_padding_and_unmeasured_rows(h):
    """|Gamma| = 18 (the cost-sorted staging kernel) with padding configs, equal costs (the
    prefix-maximum-at-group-end branch), H >= 128 so every staging buffer is reused several
    times, and whole windows unmeasured (all NaN): padding positions must stay unmeasured
    across buffer reuse, so these valid inputs keep the oracle's mask with no data error."""
    rng = np.random.default_rng(44)
    Q, n = 200, 18
    for H in (128, 130, 500):
        c = rng.choice([1.0, 2.0, 4.0], (Q, n)).astype(np.float32)   # many equal costs
        c[:, 15:] = np.inf                                            # padding positions
        A = rng.uniform(0, 1, (Q, H, n)).astype(np.float32)
        A[:, ::3, :] = np.nan                                         # unmeasured windows
        A[rng.uniform(size=A.shape) < 0.1] = np.nan
        for m in (0.0, 0.1):
            keep = ek().prune_configs(h, torch.from_numpy(c).cuda(), torch.from_numpy(A).cuda(), m)
            ok, bad = oracle.prune(c, A, m)
            assert bad == 0 and h.last_error() == 0, f"H={H}"
            assert_eq(keep, ok, f"keep mask H={H} margin={m}")


# ---------------------------------------------------------------------------
# NEXT-2: micro-profiler curve fit
# ---------------------------------------------------------------------------
def curve_inputs(S, P, seed):
    """Profile-epoch accuracies from the Optimus family plus noise (sigma 0.02),
    some constant and some degenerate sets, and the configs' full epoch counts."""
    rng = np.random.default_rng(seed)
    k = np.arange(1, P + 1, dtype=np.float64)
    b0, b1, b2 = rng.uniform(0.1, 2.0, S), rng.uniform(0.8, 3.0, S), rng.uniform(0.0, 0.3, S)
    a = 1.0 - (1.0 / (b0[:, None] * k + b1[:, None]) + b2[:, None]) + rng.normal(0, 0.02, (S, P))
    a[::7] = rng.uniform(0.2, 0.9, (len(a[::7]), 1))             # constant profiles
    a[3::11] = a[3::11, ::-1]                                      # decreasing profiles
    a = np.clip(a, 0, 1).astype(np.float32)
    K = rng.integers(P, 60, S).astype(np.int32)
    return a, K


@pytest.mark.parametrize("P", [5, 2, 9])
def test_curve_fit_bitexact(h, P):
    a, K = curve_inputs(4000, P, 60 + P)
    pred, prm = ek().curve_fit(h, torch.from_numpy(a).cuda(), torch.from_numpy(K).cuda())
    op, oprm, bad = oracle.curve_fit(a, K)
    assert bad == 0 and h.last_error() == 0
    assert_eq(pred, op, "predicted accuracy")
    assert_eq(prm, oprm, "params")


def test_curve_fit_invalid(h):
    a, K = curve_inputs(64, 5, 70)
    a[3, 2] = 1.5
    K[5] = 0
    pred, prm = ek().curve_fit(h, torch.from_numpy(a).cuda(), torch.from_numpy(K).cuda())
    op, oprm, bad = oracle.curve_fit(a, K)
    assert bad == 2 and h.last_error() == -6
    assert_eq(pred, op, "predicted accuracy")


# ---------------------------------------------------------------------------
# NEXT-1: the window timeline with re-invocation at completions
# ---------------------------------------------------------------------------
WINDOW_CASES = [("c2", variant(synth.CONFIG2, n_inst=96)),
                ("c2-ragged", variant(synth.CONFIG2, n_inst=48, ragged=True)),
                ("c1", variant(synth.CONFIG1, n_inst=300)),
                ("odd", variant(synth.CONFIG2, n_inst=24, n_streams=7, n_gamma=31, units=53, a_min=0.0)),
                ("nogamma", variant(synth.CONFIG2, n_inst=16, n_gamma=0))]


@pytest.mark.parametrize("mode", [0, 1], ids=["steepest", "literal"])
@pytest.mark.parametrize("name,cfg", WINDOW_CASES, ids=[c[0] for c in WINDOW_CASES])
def test_window_bitexact(h, name, cfg, mode):
    Td, inst = tables(cfg)
    avg, ev, done = ek().window_schedule(h, Td, *args(cfg), mode=mode)
    oavg, oev, odone, bad = oracle.window(inst, mode)
    assert bad == 0 and h.last_error() == 0
    assert_eq(ev, oev, "invocations")
    assert_eq(done, odone, "completion times")
    assert_eq(avg, oavg, "realized average")


def test_window_invalid_instance(h):
    cfg = variant(synth.CONFIG2, n_inst=8)
    T = synth.sched_tables(cfg)
    T["cost"][5, 3, 2] = -1.0
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            *args(cfg))
    avg, ev, done = ek().window_schedule(h, {k: v.cuda() for k, v in T.items()}, *args(cfg))
    oavg, oev, odone, bad = oracle.window(inst, 0)
    assert bad == 1 and h.last_error() == -6
    assert_eq(avg, oavg, "realized average")
    assert_eq(done, odone, "completion times")
