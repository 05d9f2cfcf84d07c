"""Pins for the CPU oracle (-m "not gpu").

The oracle must not be checked against itself.  Each test below compares it with
something the paper or mathematics fixes:
  * worked examples printed in SPEC.md / PAPER.md (tests/golden/*.json, cited);
  * closed forms evaluated in exact rational arithmetic (fractions.Fraction) in a
    DIFFERENT algebraic form (SPEC S:227's (t_r a_old + (T - t_r) a_new)/T rather
    than the oracle's post - f (post - stale));
  * brute force on tiny inputs written independently here from Alg. 2 / Eq. 1;
  * invariants (capacity, monotone acceptance, sandwich fair <= thief <= optimum,
    k-means fixed point, etc.);
  * a line-by-line Python transliteration of Algorithm 1's loop structure.
"""
from __future__ import annotations

import itertools
import json
import math
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ULP = 2.0 ** -23


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def f32(x):
    return float(np.float32(x))


# ---------------------------------------------------------------------------
# independent exact evaluator (Alg. 2, window average S:227)
# ---------------------------------------------------------------------------
def exact_stream(stale, costs, posts, lmus, lfs, rt, ri, uT, a_min):
    """Returns (value, gamma, lam, candidates) in exact rationals from float inputs.

    lambda pool: ri >= lam_min_units and stale*factor >= a_MIN, max accuracy.
    gamma: argmax over {none} + {gamma : t_r <= ||T||} of the window average
    (t_r a_old + (T - t_r) a_new) / T with a_old = stale*f, a_new = post*f."""
    st = Fr(stale)
    pool = [(st * Fr(lfs[l]), l) for l in range(len(lfs))
            if lmus[l] != 0xFFFF and ri >= lmus[l] and st * Fr(lfs[l]) >= Fr(a_min)]
    if not pool:
        return Fr(0), 0, 7, []
    best_acc = max(a for a, _ in pool)
    lam = min(l for a, l in pool if a == best_acc)
    fac = Fr(lfs[lam])
    T = Fr(1)  # measure time in units of ||T||: t_r/||T|| = cost / (rt * uT)
    cands = [(st * fac, 0)]
    for g in range(len(costs)):
        if rt < 1 or math.isinf(costs[g]):
            continue
        tr = Fr(costs[g]) / (rt * Fr(uT))
        if tr > T:
            continue
        a_old, a_new = st * fac, Fr(posts[g]) * fac
        cands.append(((tr * a_old + (T - tr) * a_new) / T, g + 1))
    val = max(c for c, _ in cands)
    gam = min(g for c, g in cands if c == val)
    return val, gam, lam, cands


def inst_stream(inst, b, v, rt, ri):
    return exact_stream(float(inst.stale[b, v]), [float(x) for x in inst.cost[b, v]],
                        [float(x) for x in inst.post[b, v]], [int(x) for x in inst.lam_min_units[b, v]],
                        [float(x) for x in inst.lam_factor[b, v]], rt, ri, inst.unit_gpu_seconds,
                        inst.a_min)


def boundary_case(inst, b, v, rt, ri, eps=1e-6):
    """True if an fp32-vs-exact decision (lambda filter, feasibility) sits within eps of its threshold."""
    st = float(inst.stale[b, v])
    for l in range(inst.nL):
        if ri >= inst.lam_min_units[b, v, l] and abs(st * float(inst.lam_factor[b, v, l]) - inst.a_min) < eps:
            return True
    if rt >= 1:
        for g in range(inst.nG):
            c = float(inst.cost[b, v, g])
            if not math.isinf(c) and abs(c / (rt * inst.unit_gpu_seconds) - 1.0) < eps:
                return True
    return False


def make_inst(cfg, lo=0, hi=None):
    T = synth.sched_tables(cfg, lo, hi)
    return oracle.Instances(T["stale"].numpy(), T["cost"].numpy(), T["post"].numpy(),
                            T["lam_min_units"].numpy(), T["lam_factor"].numpy(), cfg.units,
                            cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)


def table1_inst():
    fx = load("table1_fixture.json")
    uT = f32(fx["delta_gpu"] * fx["window_s"])
    return fx, oracle.Instances(np.array([fx["stale"]]), np.array([fx["cost_gpu_s"]]),
                                np.array([fx["post"]]),
                                np.array([[fx["lam_min_units"]] * 2]),
                                np.array([[fx["lam_factor"]] * 2]), fx["units"], 1, uT, fx["a_min"])


# ---------------------------------------------------------------------------
# rules 1-2: EstimateAccuracy
# ---------------------------------------------------------------------------
def test_estimator_spec_examples():
    ex = load("spec_examples.json")["estimator"]
    # gamma = NONE -> stale (factor 1): the value of a stream with Gamma = {none}
    e = ex[0]
    inst = oracle.Instances([[e["stale"]]], np.zeros((1, 1, 0)), np.zeros((1, 1, 0)), [[[1]]],
                            [[[e["factor"]]]], 4, 1, 30.0, 0.0)
    val, cfg = oracle.stream_value(inst, 0, 0, 2, 2)
    assert val == f32(e["expect"]) and cfg == 0
    # T=120, t_r=60 -> f = 0.5; with one unit = 1 GPU, uT = 120, cost = 60 GPU-s
    e = ex[1]
    g = oracle.window_accuracy(e["a_old"], e["a_new"], e["t_r"], 1, e["window_s"])
    assert f32(g) == f32(e["expect"])
    # t_r = 130 > 120 -> infeasible
    e = ex[2]
    assert not oracle.gamma_feasible(e["t_r"], 1, e["window_s"])
    assert oracle.gamma_feasible(e["window_s"], 1, e["window_s"])  # t_r == ||T|| is feasible (C5)


def test_retrain_duration_spec_examples():
    # t_r = cost / (rt * delta); with delta = 0.5 GPU and ||T|| = 200 s, uT = 100 GPU-s/unit
    delta, T = 0.5, 200.0
    for e in load("spec_examples.json")["retrain_duration"]:
        cost = e["epochs"] * e["gpu_s_per_epoch"] * e["data_fraction"]   # P:1155 scaling
        rt = int(round(e["share"] / delta))
        f = oracle.retrain_fraction(cost, rt, delta * T)
        assert f32(f * T) == pytest.approx(e["expect_s"], rel=1e-6), e["cite"]


def test_estimator_vs_exact_closed_form():
    rng = np.random.default_rng(1)
    for _ in range(4000):
        stale, post = f32(rng.uniform(0, 1)), f32(rng.uniform(0, 1))
        uT = f32(rng.uniform(1, 50))
        rt = int(rng.integers(1, 100))
        cost = f32(rng.uniform(0, rt * uT))
        if not oracle.gamma_feasible(cost, rt, uT):
            continue
        g = oracle.window_accuracy(stale, post, cost, rt, uT)
        tr = Fr(cost) / (rt * Fr(uT))
        exact = tr * Fr(stale) + (1 - tr) * Fr(post)        # draft P:73 at t = 0
        assert abs(Fr(g) - exact) <= Fr(4 * ULP), (stale, post, cost, rt, uT)


def test_estimator_monotone_in_rt():
    """North star invariant: accuracy is monotone in r_train for fixed gamma
    (non-decreasing if post >= stale, non-increasing otherwise)."""
    rng = np.random.default_rng(2)
    for _ in range(300):
        stale, post = f32(rng.uniform(0, 1)), f32(rng.uniform(0, 1))
        uT, cost = f32(rng.uniform(1, 30)), f32(rng.uniform(0, 2000))
        prev, seen = None, False
        for rt in range(1, 300):
            feas = oracle.gamma_feasible(cost, rt, uT)
            if not feas:
                assert not seen, "feasibility must be an up-set in rt"
                continue
            seen = True
            g = oracle.window_accuracy(stale, post, cost, rt, uT)
            if prev is not None:
                assert (g >= prev) if post >= stale else (g <= prev)
            prev = g


def test_q32_rounding():
    assert oracle.q32(0.0) == 0
    assert oracle.q32(1.0) == 2 ** 32
    assert oracle.q32(0.5) == 2 ** 31
    assert oracle.q32(2.0 ** -33) == 0          # 0.5 -> nearest even
    assert oracle.q32(3 * 2.0 ** -33) == 2      # 1.5 -> 2
    assert oracle.q32(5 * 2.0 ** -33) == 2      # 2.5 -> 2
    x = f32(0.7)
    assert oracle.q32(x) == round(Fr(x) * 2 ** 32)


# ---------------------------------------------------------------------------
# rule 3: PickConfigs
# ---------------------------------------------------------------------------
def test_pickconfigs_vs_exact_enumeration():
    for cfg, n in ((synth.CONFIG1, 60), (synth.CONFIG2, 6)):
        cfgr = synth.SchedConfig(**{**cfg.__dict__, "ragged": True}) if cfg is synth.CONFIG2 else cfg
        for c in (cfg, cfgr):
            inst = make_inst(c, 0, n)
            rng = np.random.default_rng(3)
            for b in range(inst.B):
                for _ in range(6):
                    rt = rng.integers(0, inst.units + 1, inst.V)
                    ri = rng.integers(0, inst.units + 1, inst.V)
                    alloc = np.stack([ri, rt], 1).reshape(-1)
                    s, cfgs, vals = oracle.pickconfigs(inst, b, alloc)
                    tot = 0
                    for v in range(inst.V):
                        if boundary_case(inst, b, v, int(rt[v]), int(ri[v])):
                            continue
                        ev, eg, el, cands = inst_stream(inst, b, v, int(rt[v]), int(ri[v]))
                        assert abs(Fr(float(vals[v])) - ev) <= Fr(1, 10 ** 6)
                        assert (cfgs[v] >> 5) == el
                        others = sorted((c for c, g in cands if g != eg), reverse=True)
                        if not others or ev - others[0] > Fr(1, 10 ** 6):
                            assert (cfgs[v] & 31) == eg
                        tot += oracle.q32(float(vals[v]))
                    assert s >= 0


def test_pickconfigs_gamma_empty_special_case():
    """Gamma = {none} -> no retraining, value = best feasible lambda accuracy."""
    inst = oracle.Instances([[0.8, 0.6]], np.zeros((1, 2, 0)), np.zeros((1, 2, 0)),
                            [[[3, 1], [2, 1]]], [[[1.0, 0.5], [0.9, 0.8]]], 10, 1, 20.0, 0.41)
    s, cfg, vals = oracle.pickconfigs(inst, 0, [3, 7, 1, 0])
    assert vals[0] == f32(0.8) and cfg[0] == 0                       # lambda 0, no gamma
    assert vals[1] == f32(f32(0.6) * f32(0.8)) and cfg[1] == (1 << 5)  # lambda 1 (lambda 0 needs 2 units)
    s, cfg, vals = oracle.pickconfigs(inst, 0, [2, 0, 0, 8])
    # stream 0 at ri = 2: lambda 0 needs 3 units, lambda 1 gives 0.4 < a_MIN 0.41 -> none (C8)
    assert vals[0] == 0.0 and (cfg[0] >> 5) == 7
    assert vals[1] == 0.0 and (cfg[1] >> 5) == 7


def test_pickconfigs_exact_ties_and_amin_boundary():
    """C7 (Alg. 2's strict '>' from best_accuracy): on exact ties the lowest
    index wins, for gamma (no retraining first) and for lambda; C3: a lambda whose accuracy
    equals a_MIN exactly is admissible (">= a_MIN").  uT = 20, a_MIN = 0.4.
      stream 0: stale 0.5, lambdas factor 0.875 twice (both need 1 unit) -> lambda 0;
                configs 0 and 1 identical (cost 10, post 0.8): at r_train 1, f = 1/2,
                value 0.875 (0.8 - 0.5 * 0.3) = 0.56875 for both -> gamma 1 (index 0 + 1).
      stream 1: stale 0.6, one config with post = stale (cost 5): its window value equals
                the stale model's -> no retraining (gamma 0); lambda 1 (factor 1.0) needs
                3 units, so at r_infer 2 lambda 0 (factor 0.75, value 0.45).
      stream 2: stale 0.5, lambda factor 0.8: accuracy 0.5 * 0.8 = 0.4 = a_MIN exactly
                (both binary32 0.4f) -> admissible, value 0.4; no real config (padding)."""
    inf = float("inf")
    inst = oracle.Instances([[0.5, 0.6, 0.5]],
                            [[[10.0, 10.0], [5.0, inf], [inf, inf]]],
                            [[[0.8, 0.8], [0.6, 0.0], [0.0, 0.0]]],
                            [[[1, 1], [1, 3], [1, 0xFFFF]]],
                            [[[0.875, 0.875], [0.75, 1.0], [0.8, 1.0]]], 12, 1, 20.0, 0.4)
    assert np.float32(0.5) * np.float32(0.8) == np.float32(0.4)
    s, cfg, vals = oracle.pickconfigs(inst, 0, [2, 1, 2, 1, 1, 0])
    assert cfg.tolist() == [1, 0, 0]
    assert vals[0] == np.float32(0.875) * np.float32(np.float32(0.8) - np.float32(0.5) * (np.float32(0.8) -
                                                                                         np.float32(0.5)))
    assert vals[0] == pytest.approx(0.56875, abs=1e-7)
    assert vals[1] == np.float32(0.75) * np.float32(0.6)
    assert vals[2] == np.float32(0.4)
    # the same choices through a LIST row and a GRID cell of stream 0
    ls, lm, lc, bad = oracle.eval_list(inst, np.array([[[2, 1, 2, 1, 1, 0]]], np.uint16))
    assert bad == 0 and lc[0, 0].tolist() == [1, 0, 0]


def test_table1_uniform_inference_accuracy():
    """at 0.75 GPU each, inference accuracy drops 65% -> 49% and 50% -> 37.5%."""
    fx, inst = table1_inst()
    e = fx["expect"]["uniform_inference_accuracy"]
    nog = oracle.Instances(inst.stale, np.zeros((1, 2, 0)), np.zeros((1, 2, 0)),
                           inst.lam_min_units, inst.lam_factor, inst.units, 1, inst.unit_gpu_seconds, 0.0)
    a, _ = oracle.stream_value(nog, 0, 0, 0, e["ri_units"])
    b, _ = oracle.stream_value(nog, 0, 1, 0, e["ri_units"])
    assert a == pytest.approx(e["A"], abs=e["tol"])
    assert b == pytest.approx(e["B"], abs=e["tol"])


def test_fair_allocation_rule():
    """C9: equal per-stream split (remainder to low streams), floor half to retraining."""
    for V, U in ((10, 80), (3, 10), (2, 10), (7, 5), (1, 1)):
        inst = oracle.Instances(np.full((1, V), 0.5), np.zeros((1, V, 0)), np.zeros((1, V, 0)),
                                np.ones((1, V, 1)), np.ones((1, V, 1)), U, 1, 10.0, 0.0)
        a = oracle.fair(inst)
        assert a.sum() == U
        shares = a[0::2] + a[1::2]
        assert shares.max() - shares.min() <= 1 and list(shares) == sorted(shares, reverse=True)
        assert all(a[1::2] == shares // 2)
    inst = oracle.Instances(np.full((1, 3), 0.5), np.zeros((1, 3, 0)), np.zeros((1, 3, 0)),
                            np.ones((1, 3, 1)), np.ones((1, 3, 1)), 10, 1, 10.0, 0.0)
    assert list(oracle.fair(inst)) == [2, 2, 2, 1, 2, 1]


# ---------------------------------------------------------------------------
# LIST / GRID evaluators
# ---------------------------------------------------------------------------
def test_eval_list_matches_exact_and_flags_invalid_rows():
    inst = make_inst(synth.CONFIG2, 0, 3)
    rows = synth.list_allocs(synth.CONFIG2, 8, 0, 3).numpy().astype(np.uint16)
    assert (rows.astype(np.int64).sum(-1) == inst.units).all()
    rows[1, 0, 0] = inst.units + 1            # entry > U
    rows[2, 1, 3] += 5                        # sum > U
    s, mean, cfg, bad = oracle.eval_list(inst, rows)
    assert bad == 2 and s[1, 0] == 0 and s[2, 1] == 0 and mean[1, 0] == 0.0
    for b in range(3):
        for n in range(8):
            if (b, n) in ((1, 0), (2, 1)):
                continue
            tot = Fr(0)
            for v in range(inst.V):
                ev, *_ = inst_stream(inst, b, v, int(rows[b, n, 2 * v + 1]), int(rows[b, n, 2 * v]))
                tot += ev
            assert abs(Fr(int(s[b, n]), 2 ** 32) - tot) <= Fr(inst.V, 10 ** 6)
            assert mean[b, n] == oracle.mean_from_q32(int(s[b, n]), inst.V)


def test_eval_grid_cells_and_ri_monotone():
    inst = make_inst(synth.CONFIG1, 0, 20)
    grid, gcfg, bad = oracle.eval_grid(inst)
    assert bad == 0
    U = inst.units
    for b in range(inst.B):
        for v in range(inst.V):
            c = 0
            for rt in range(U + 1):
                row = grid[b, v, c:c + U + 1 - rt]
                assert (np.diff(row) >= 0).all()      # lambda pool grows with ri
                for ri in range(U + 1 - rt):
                    if not boundary_case(inst, b, v, rt, ri):
                        ev, eg, el, _ = inst_stream(inst, b, v, rt, ri)
                        assert abs(Fr(float(grid[b, v, c + ri])) - ev) <= Fr(1, 10 ** 6)
                c += U + 1 - rt


# ---------------------------------------------------------------------------
# Eq. 1 brute force
# ---------------------------------------------------------------------------
def test_bruteforce_vs_exact_exhaustive():
    inst = make_inst(synth.CONFIG1, 0, 12)
    alloc, cfg, s, bad = oracle.bruteforce(inst)
    U, J = inst.units, 2 * inst.V
    for b in range(inst.B):
        best = Fr(-1)
        vals = {}
        for comp in itertools.product(range(U + 1), repeat=J):
            if sum(comp) > U:
                continue
            tot = sum(inst_stream(inst, b, v, comp[2 * v + 1], comp[2 * v])[0] for v in range(inst.V))
            vals[comp] = tot
            best = max(best, tot)
        got = vals[tuple(int(x) for x in alloc[b])]
        assert best - got <= Fr(inst.V, 10 ** 6)
        assert abs(Fr(int(s[b]), 2 ** 32) - best) <= Fr(inst.V, 10 ** 6)


def test_table1_optimum_qualitative():
    fx, inst = table1_inst()
    alloc, cfg, s, _ = oracle.bruteforce(inst)
    e = fx["expect"]
    assert (cfg[0, e["optimum_picks_cheaper_cfg_for_B"]["stream"]] & 31) == \
        e["optimum_picks_cheaper_cfg_for_B"]["gamma_index"]           # Cfg2B
    assert alloc[0, 3] > alloc[0, 1]                                  # rt_B > rt_A
    fair = oracle.fair(inst)
    sf, _, _ = oracle.pickconfigs(inst, 0, fair)
    assert int(s[0]) > sf
    # the STEEPEST thief reaches the same qualitative decision on this instance
    ta, tc, ts, *_ = oracle.thief(inst, oracle.STEEPEST)
    assert (tc[0, 1] & 31) == 2 and ta[0, 3] > ta[0, 1]


# ---------------------------------------------------------------------------
# Algorithm 1: structure + invariants
# ---------------------------------------------------------------------------
def py_literal(inst, b):
    """Algorithm 1 transliterated line by line; objective = oracle PickConfigs."""
    J, D = 2 * inst.V, inst.steal_units
    pick = lambda a: oracle.pickconfigs(inst, b, a)[0]
    best = list(oracle.fair(inst))                       # line 2
    best_acc = pick(best)                                # line 3
    for thief in range(J):                               # line 5
        for victim in range(J):                          # line 6
            if thief == victim:                          # line 7
                continue
            temp = list(best)                            # line 8
            while True:                                  # line 9
                temp[victim] -= D                        # line 10
                temp[thief] += D                         # line 11
                if temp[victim] < 0:                     # line 12
                    break
                acc = pick(temp)                         # line 14
                if acc > best_acc:                       # line 15
                    best, best_acc = list(temp), acc     # lines 16-18
                else:
                    break                                # line 20
    return best, best_acc


def py_steepest(inst, b):
    J, D = 2 * inst.V, inst.steal_units
    pick = lambda a: oracle.pickconfigs(inst, b, a)[0]
    a = list(oracle.fair(inst))
    cur, steps = pick(a), 0
    while True:
        cands = []
        for t in range(J):
            for w in range(J):
                if t != w and a[w] >= D:
                    x = list(a)
                    x[w] -= D
                    x[t] += D
                    cands.append((-pick(x), t, w))
        best = min(cands)
        if -best[0] <= cur:
            return a, cur, steps
        a[best[2]] -= D
        a[best[1]] += D
        cur, steps = -best[0], steps + 1


@pytest.mark.parametrize("cfg,n", [(synth.CONFIG1, 40), (synth.CONFIG2, 3)])
def test_thief_matches_transliteration(cfg, n):
    inst = make_inst(cfg, 0, n)
    la, _, ls, _, lsteps, _ = oracle.thief(inst, oracle.LITERAL)
    sa, _, ss, _, ssteps, _ = oracle.thief(inst, oracle.STEEPEST)
    for b in range(n):
        pa, ps = py_literal(inst, b)
        assert list(la[b]) == pa and int(ls[b]) == ps
        qa, qs, qsteps = py_steepest(inst, b)
        assert list(sa[b]) == qa and int(ss[b]) == qs and int(ssteps[b]) == qsteps


def test_thief_invariants_and_sandwich():
    cfg = synth.SchedConfig(**{**synth.CONFIG1.__dict__, "n_inst": 1500})
    inst = make_inst(cfg)
    U, J = inst.units, 2 * inst.V
    ba, _, bs, _ = oracle.bruteforce(inst)
    fair = oracle.fair(inst)
    for mode in (oracle.STEEPEST, oracle.LITERAL):
        a, c, s, mean, steps, bad = oracle.thief(inst, mode)
        assert bad == 0
        assert (a.astype(np.int64).sum(1) == U).all()                      # P:1120 capacity
        for b in range(inst.B):
            sf = oracle.pickconfigs(inst, b, fair)[0]
            assert sf <= int(s[b]) <= int(bs[b])                           # S:289 sandwich
            assert (steps[b] == 0) == (int(s[b]) == sf)                     # strict acceptance
            assert steps[b] <= J * J * U // inst.steal_units               # S:288 bound
            assert mean[b] == oracle.mean_from_q32(int(s[b]), inst.V)
    # STEEPEST stops at a point no single Delta-steal improves
    a, c, s, *_ = oracle.thief(inst.subset(range(200)), oracle.STEEPEST)
    for b in range(200):
        for t in range(J):
            for w in range(J):
                if t != w and a[b, w] >= 1:
                    x = a[b].astype(np.int32).copy()
                    x[w] -= 1
                    x[t] += 1
                    assert oracle.pickconfigs(inst, b, x)[0] <= int(s[b])


def test_invalid_instance_is_zeroed():
    inst = make_inst(synth.CONFIG1, 0, 3)
    inst.cost[1, 0, 0] = -1.0
    inst.stale[2, 1] = float("nan")
    a, c, s, mean, steps, bad = oracle.thief(inst, oracle.STEEPEST)
    assert bad == 2 and (a[1:] == 0).all() and (s[1:] == 0).all() and s[0] > 0


# ---------------------------------------------------------------------------
# profiler
# ---------------------------------------------------------------------------
def test_profile_spec_examples():
    ex = load("spec_examples.json")
    for e in ex["distance"]:
        # distance <= tau exactly at the printed distance (one-window history, acc 0.5)
        d = e["expect"]
        for tau, hit in ((d * (1 + 1e-6) + 1e-9, True), (d * (1 - 1e-6) - 1e-9, False)):
            if tau < 0:
                continue
            est, n, _, _ = oracle.profile([e["p"]], [[e["q"]]], [[[0.5]]], [[0.1]], tau=tau)
            assert (n[0, 0] == 1) == hit, e["cite"]
    for e in ex["history_estimate"]:
        est, n, _, _ = oracle.profile([e["cur"]], [e["hist"]], [[[a] for a in e["acc"]]], [[-1.0]],
                                      tau=e["tau"])
        if e["expect"] == "absent":
            assert n[0, 0] == 0 and est[0, 0] == f32(-1.0), e["cite"]
        else:
            assert est[0, 0] == pytest.approx(e["expect"], abs=1e-7), e["cite"]


def test_profile_radius_inclusive_at_exact_boundary():
    """C17: similar iff d <= tau, inclusive.  cur (0.5, 0.5) vs window (0.5, 0.25):
    every operation of rule 5 is exact here (d^2 = 0 + 0.0625, sqrt = 0.25), so at
    tau = 0.25 the window is similar and at the next binary32 below 0.25 it is not.  Also
    in CLUSTER's join and every other profile path tau is the only threshold, so this is
    the whole boundary behaviour."""
    below = float(np.nextafter(np.float32(0.25), np.float32(0.0)))
    for tau, hit in ((0.25, True), (below, False), (0.0, False)):
        est, n, _, bad = oracle.profile([[0.5, 0.5]], [[[0.5, 0.25]]], [[[0.625]]], [[0.125]], tau=tau)
        assert bad == 0
        assert n[0, 0] == (1 if hit else 0)
        assert est[0, 0] == (np.float32(0.625) if hit else np.float32(0.125))
    # a window at distance exactly 0 is similar even at tau = 0
    est, n, _, _ = oracle.profile([[0.5, 0.5]], [[[0.5, 0.5]]], [[[0.625]]], [[0.125]], tau=0.0)
    assert n[0, 0] == 1 and est[0, 0] == np.float32(0.625)


@pytest.mark.parametrize("sparse", [False, True])
def test_profile_radius_vs_float64_bruteforce(sparse):
    cfg = synth.ProfileConfig("t", 24, 300, 27, 18, sparse=sparse)
    P = {k: v.numpy() for k, v in synth.profile_inputs(cfg).items()}
    est, n, _, bad = oracle.profile(P["cur"], P["hist"], P["hist_acc"], P["fallback"], tau=0.2)
    assert bad == 0
    d = np.sqrt(((P["hist"].astype(np.float64) - P["cur"][:, None, :]) ** 2).sum(-1))
    for q in range(cfg.n_query):
        if np.any(np.abs(d[q] - 0.2) < 1e-5):
            continue
        sim = d[q] <= 0.2
        for g in range(cfg.n_gamma):
            a = P["hist_acc"][q, :, g].astype(np.float64)
            m = sim & ~np.isnan(a)
            assert n[q, g] == m.sum()
            if m.sum():
                assert est[q, g] == pytest.approx(a[m].mean(), abs=1e-7)
            else:
                assert est[q, g] == P["fallback"][q, g]


def test_cluster_recovers_separated_clusters_and_fixed_point():
    rng = np.random.default_rng(5)
    Q, H, C, K = 6, 200, 8, 5
    hist = np.zeros((Q, H, C), np.float32)
    truth = np.zeros((Q, H), np.int64)
    for q in range(Q):
        lab = rng.integers(0, K, H)
        lab[[i * H // K for i in range(K)]] = rng.permutation(K)   # C19 init points in distinct clusters
        truth[q] = lab
        for h in range(H):
            x = np.full(C, 0.01)
            x[lab[h]] = 1.0                     # one dominant class per cluster
            x = x + rng.uniform(0, 0.02, C)
            hist[q, h] = x / x.sum()
    acc = rng.uniform(0.3, 0.9, (Q, H, 3)).astype(np.float32)
    cur = hist[:, 7, :].copy()
    est, n, cl, bad = oracle.profile(cur, hist, acc, np.zeros((Q, 3)), mode=oracle.CLUSTER, k=K)
    for q in range(Q):
        a = cl[q, :H]
        # same partition as the ground truth (labels may be permuted)
        pairs = set(zip(a.tolist(), truth[q].tolist()))
        assert len(pairs) == K and len({p[0] for p in pairs}) == K
        # fixed point in float64: every window is nearest its own cluster mean
        mu = np.stack([hist[q][a == i].astype(np.float64).mean(0) for i in range(K)])
        dd = ((hist[q][:, None, :].astype(np.float64) - mu[None]) ** 2).sum(-1)
        assert (dd[np.arange(H), a] <= dd.min(1) + 1e-9).all()
        # query joins the nearest centroid; estimate = mean accuracy over that cluster
        assert cl[q, H] == a[7]
        m = a == cl[q, H]
        assert n[q, 0] == m.sum()
        assert est[q, 0] == pytest.approx(acc[q, m, 0].astype(np.float64).mean(), abs=1e-7)


def test_cluster_degenerate_identical_histograms():
    H = 50
    hist = np.tile(np.array([0.2, 0.3, 0.5], np.float32), (1, H, 1))
    acc = np.linspace(0.1, 0.9, H, dtype=np.float32).reshape(1, H, 1)
    est, n, cl, _ = oracle.profile(hist[:, 0], hist, acc, [[0.0]], mode=oracle.CLUSTER, k=5)
    assert (cl[0] == 0).all() and n[0, 0] == H
    assert est[0, 0] == pytest.approx(acc.astype(np.float64).mean(), abs=1e-7)


def _hist2(xs):
    """Two-class histograms (x, 1 - x); every value below is a multiple of 1/16, so the
    coordinates, their differences and squares are exact in binary32."""
    return np.array([[[x, 1.0 - x] for x in xs]], np.float32)


def test_cluster_init_and_ties_hand_worked():
    """C19 initial centroids mu_i = h_floor(iH/k) and lowest index on distance ties.
    H = 4 windows x = 1/16, 9/16, 3/4, 5/16 (histograms (x, 1-x)), k = 3:
      init mu = (h_0, h_1, h_2) = (1/16, 9/16, 3/4)   [floor(4/3) = 1, floor(8/3) = 2];
      assign: 5/16 is equidistant (1/4) from 1/16 and 9/16 -> lowest index 0:
              (0, 1, 2, 0);
      update: mu_0 = (1/16 + 5/16)/2 = 3/16, mu_1 = 9/16, mu_2 = 3/4;
      reassign: unchanged -> stop.  Final (0, 1, 2, 0).
    (A ceil(iH/k) init, mu = (1/16, 3/4, 5/16), converges to (0, 1, 1, 2) instead.)
    The query (3/16, 13/16) joins cluster 0: estimate = mean of windows 0 and 3."""
    hist = _hist2([1 / 16, 9 / 16, 3 / 4, 5 / 16])
    acc = np.array([[[0.25], [0.5], [0.75], [0.5]]], np.float32)
    est, n, cl, bad, passes = oracle.profile(_hist2([3 / 16])[:, 0], hist, acc, [[0.0]], mode=oracle.CLUSTER, k=3,
                                             with_passes=True)
    assert bad == 0
    assert passes.tolist() == [2]          # the initial assignment + one iteration (no change)
    assert cl[0].tolist() == [0, 1, 2, 0, 0]
    assert n[0, 0] == 2 and est[0, 0] == np.float32(0.375)


def test_cluster_empty_cluster_keeps_its_centroid():
    """C19 "empty cluster keeps its centroid", hand-worked.  H = 7 windows
    x = 11/16, 13/16, 11/16, 0, 5/8, 7/8, 0 (histograms (x, 1-x)), k = 3:
      init mu = (h_0, h_2, h_4) = (11/16, 11/16, 5/8);
      assign (ties to the lowest index, so cluster 1 -- a copy of centroid 0 -- gets
              nobody): (0, 0, 0, 2, 2, 0, 2);
      update: mu_0 = (11+13+11+14)/64 = 49/64, mu_1 = 11/16 KEPT (empty), mu_2 = 5/24;
      assign: 11/16 -> mu_1 (distance 0), 13/16 -> mu_0, 5/8 -> mu_1 (1/16 vs 9/64),
              7/8 -> mu_0, 0 -> mu_2: (1, 0, 1, 2, 1, 0, 2);
      update: mu_0 = 27/32, mu_1 = 2/3, mu_2 = 0;  assign: unchanged -> stop.
    The query (11/16, 5/16) joins cluster 1 = windows {0, 2, 4}."""
    hist = _hist2([11 / 16, 13 / 16, 11 / 16, 0.0, 5 / 8, 7 / 8, 0.0])
    acc = np.array([[[0.5], [0.1], [0.75], [0.2], [1.0], [0.3], [0.4]]], np.float32)
    est, n, cl, bad, passes = oracle.profile(_hist2([11 / 16])[:, 0], hist, acc, [[0.0]], mode=oracle.CLUSTER, k=3,
                                             with_passes=True)
    assert bad == 0
    assert passes.tolist() == [3]          # initial + two iterations (the second changes nothing)
    assert cl[0].tolist() == [1, 0, 1, 2, 1, 0, 2, 1]
    assert n[0, 0] == 3 and est[0, 0] == np.float32(0.75)
    # max_iter bounds the iterations: with one, the first update's assignment is final; with
    # none, the initial assignment is (the query then joins cluster 0, tied with cluster 1)
    _, _, cl1, _, p1 = oracle.profile(_hist2([11 / 16])[:, 0], hist, acc, [[0.0]], mode=oracle.CLUSTER, k=3,
                                      max_iter=1, with_passes=True)
    assert p1.tolist() == [2] and cl1[0].tolist() == [1, 0, 1, 2, 1, 0, 2, 1]
    _, n0, cl0, _, p0 = oracle.profile(_hist2([11 / 16])[:, 0], hist, acc, [[0.0]], mode=oracle.CLUSTER, k=3,
                                       max_iter=0, with_passes=True)
    assert p0.tolist() == [1] and cl0[0].tolist() == [0, 0, 0, 2, 2, 0, 2, 0] and n0[0, 0] == 4


def test_cluster_on_synth_converges_to_fixed_point():
    cfg = synth.ProfileConfig("t", 8, 500, 27, 18)
    P = {k: v.numpy() for k, v in synth.profile_inputs(cfg).items()}
    est, n, cl, bad = oracle.profile(P["cur"], P["hist"], P["hist_acc"], P["fallback"],
                                     mode=oracle.CLUSTER, k=5, max_iter=100)
    for q in range(cfg.n_query):
        a = cl[q, :500]
        present = [i for i in range(5) if (a == i).any()]
        mu = {i: P["hist"][q][a == i].astype(np.float64).mean(0) for i in present}
        for h in range(500):
            d = {i: ((P["hist"][q, h] - mu[i]) ** 2).sum() for i in present}
            assert d[a[h]] <= min(d.values()) + 1e-6


# ---------------------------------------------------------------------------
# NEXT-4: placement onto GPUs and checkpointing
# ---------------------------------------------------------------------------
def test_quantize_spec_examples():
    """0.5 -> 0.5, 0.3 -> 0.25, 1.0 -> 1.0 (a whole GPU)."""
    Q = oracle.Q_ONE
    assert oracle.quantize_frac(5, 10) == Q // 2
    assert oracle.quantize_frac(3, 10) == Q // 4
    pj, pq, pg, npc, load, bad = oracle.place(np.array([[10]], np.uint16), 10, 1)
    assert npc[0] == 1 and pq[0, 0] == Q and pg[0, 0] == 0 and bad == 0


def test_quantize_is_largest_inverse_power_of_two_below():
    """Exact-rational definition: 2^-k <= r/U < 2^-(k-1), k >= 1, for every r < U."""
    from fractions import Fraction
    rng = np.random.default_rng(11)
    for U in [1, 2, 3, 7, 10, 80, 800, 65534]:
        for r in set(list(range(1, min(U, 40))) + list(rng.integers(1, max(2, U), 40))):
            if not 0 < r < U:
                continue
            q = Fraction(oracle.quantize_frac(int(r), U), oracle.Q_ONE)
            x = Fraction(int(r), U)
            assert q <= x < 2 * q and q.numerator == 1 and (q.denominator & (q.denominator - 1)) == 0


def test_pack_spec_examples():
    """S:337-339 (first-fit decreasing)."""
    Q = oracle.Q_ONE
    g, load = oracle.pack(np.array([Q // 2] * 4), 2)
    assert sorted(g.tolist()) == [0, 0, 1, 1] and load.tolist() == [Q, Q]
    g, load = oracle.pack(np.array([Q // 2, Q // 4, Q // 4, Q // 4, Q // 4, Q // 2]), 2)
    assert (g >= 0).all() and load.tolist() == [Q, Q]
    g, load = oracle.pack(np.array([Q, Q, Q // 2]), 2)
    assert g.tolist() == [0, 1, -1]


def test_pack_invariants_fuzzed():
    """Per-GPU load <= 1 GPU; every unplaced piece fits no GPU's final free space; with
    power-of-two pieces whose total fits, first-fit decreasing places all of them."""
    Q = oracle.Q_ONE
    rng = np.random.default_rng(12)
    for _ in range(300):
        n, G = int(rng.integers(1, 30)), int(rng.integers(1, 9))
        q = (Q >> rng.integers(0, 8, n)).astype(np.uint32)
        g, load = oracle.pack(q, G)
        assert (load <= Q).all()
        for i in np.flatnonzero(g < 0):
            assert (load + q[i] > Q).all()
        for gg in range(G):
            assert load[gg] == q[g == gg].sum()
        if q.sum() <= G * Q:
            assert (g >= 0).all()


def test_place_pieces_follow_pl1():
    """PL1 exactly (fractions): floor(a G / U) whole GPUs plus the remainder quantized down;
    total quantized <= total share; everything placed when sum a <= U (power-of-two pieces)."""
    from fractions import Fraction
    rng = np.random.default_rng(13)
    for _ in range(200):
        J, U, G = int(rng.integers(1, 24)), int(rng.integers(1, 200)), int(rng.integers(1, 12))
        w = rng.integers(0, 5, J)
        a = np.floor(w / max(1, w.sum()) * U).astype(np.uint16)
        pj, pq, pg, npc, load, bad = oracle.place(a[None, :], U, G)
        assert bad == 0
        n = int(npc[0])
        assert n <= J + G and (pg[0, :n] >= 0).all()
        for j in range(J):
            share = Fraction(int(a[j]) * G, U)
            got = [Fraction(int(x), oracle.Q_ONE) for x in pq[0, :n][pj[0, :n] == j]]
            whole = [x for x in got if x == 1]
            frac = [x for x in got if x < 1]
            assert len(whole) == int(share)
            rem = share - int(share)
            assert len(frac) == (1 if rem > 0 else 0)
            if frac:
                assert frac[0] <= rem < 2 * frac[0]
        assert sum(int(x) for x in pq[0, :n]) <= sum(int(x) for x in a) * G * oracle.Q_ONE // U + 1
    pj, pq, pg, npc, load, bad = oracle.place(np.array([[9, 9]], np.uint16), 16, 2)
    assert bad == 1 and npc[0] == 0                    # sum > U: data error


def test_checkpoint_spec_examples():
    """S:347-349."""
    out, bad = oracle.checkpoint([30], [20], [100], [0.5], [0.6], [0.9], [0.0])
    assert out[0] == 1 and bad == 0                    # free checkpoint with any gain
    out, bad = oracle.checkpoint([30], [20], [100], [0.5], [0.6], [0.9], [2.0])
    assert out[0] == 0                                 # 10 * 0.1 = 1.0 > 1.8 is false
    out, bad = oracle.checkpoint([30], [20], [100], [0.7], [0.7], [0.9], [0.5])
    assert out[0] == 0                                 # a* = a, positive cost


def test_checkpoint_exact_tie_keeps_training():
    """CK1 is strict (checkpoint iff acc > base_acc): with (tau - t)(a* - a) equal to
    delta A exactly (10 x 0.125 = 2.5 x 0.5 = 1.25, all exact in binary32) the two averaged
    accuracies are equal as rationals, so there is no checkpoint; a hair more gain tips it."""
    out, bad = oracle.checkpoint([30], [20], [100], [0.5], [0.625], [0.5], [2.5])
    assert bad == 0 and out[0] == 0
    out, bad = oracle.checkpoint([30], [20], [100], [0.5], [np.nextafter(np.float32(0.625), np.float32(1))],
                                 [0.5], [2.5])
    assert out[0] == 1


def test_checkpoint_matches_the_averaged_accuracy_form():
    """acc > base_acc in exact rationals agrees with the oracle's simplified form
    wherever the two sides differ by more than 1e-5 (rounding can only flip near ties)."""
    from fractions import Fraction as F
    rng = np.random.default_rng(14)
    n = 4000
    T = rng.uniform(10, 300, n).astype(np.float32)
    tau = (T * rng.uniform(0, 1, n)).astype(np.float32)
    t = (tau * rng.uniform(0, 1, n)).astype(np.float32)
    a, ast, A = (rng.uniform(0, 1, n).astype(np.float32) for _ in range(3))
    dl = rng.uniform(0, 20, n).astype(np.float32)
    out, bad = oracle.checkpoint(tau, t, T, a, ast, A, dl)
    assert bad == 0
    for i in range(n):
        Ti, ti, taui = F(float(T[i])), F(float(t[i])), F(float(tau[i]))
        base = ((taui - ti) * F(float(a[i])) + (Ti - taui) * F(float(A[i]))) / Ti
        acc = ((taui - ti) * F(float(ast[i])) + (Ti - taui - F(float(dl[i]))) * F(float(A[i]))) / Ti
        if abs(acc - base) > F(1, 100000):
            assert out[i] == (acc > base)
    out, bad = oracle.checkpoint([10], [20], [100], [0.5], [0.6], [0.9], [1.0])
    assert bad == 1 and out[0] == 0                    # t > tau: data error


# ---------------------------------------------------------------------------
# NEXT-3: uniform baseline and Pareto frontier
# ---------------------------------------------------------------------------
def test_uniform_allocation_spec_example():
    """2 streams, 3 GPUs, weight 0.5 -> each job gets 0.75 GPU (3 units of 0.25)."""
    fx, inst = table1_inst()
    a, cfg, s, mean, bad = oracle.uniform(inst, oracle.HIGHEST_POST, 0.5)
    assert bad == 0 and a.tolist() == [[3, 3, 3, 3]]
    assert (a[0] * fx["delta_gpu"] == 0.75).all()


def test_uniform_table1_picks_highest_accuracy_configs():
    """the baseline always retrains with the highest-accuracy configuration
    (Cfg1A, Cfg1B); at 0.75 GPU inference keeps the lambda with factor 0.75 (65% ->
    49%, 50% -> 37.5%, below the fixture's a_MIN, so a_MIN = 0 as in the P:765 pin)."""
    fx, inst0 = table1_inst()
    inst = oracle.Instances(inst0.stale, inst0.cost, inst0.post, inst0.lam_min_units, inst0.lam_factor,
                            inst0.units, 1, inst0.unit_gpu_seconds, 0.0)
    a, cfg, s, mean, bad = oracle.uniform(inst)
    assert [(c & 31) for c in cfg[0]] == [1, 1]          # config index 0 of each stream (Cfg1*)
    assert [(c >> 5) for c in cfg[0]] == [1, 1]           # lambda with factor 0.75
    # value = fl(0.75 g(Cfg1, rt = 3)) per stream, g the window average of rule 2 (pinned above)
    val = [f32(f32(0.75) * f32(oracle.window_accuracy(fx["stale"][v], fx["post"][v][0],
                                                       fx["cost_gpu_s"][v][0], 3, inst.unit_gpu_seconds)))
           for v in range(2)]
    assert int(s[0]) == sum(oracle.q32(x) for x in val)
    # both finish inside the window (85/90 and 80/90 of it), so both beat the stale model
    assert val[0] > f32(0.75 * fx["stale"][0]) and val[1] > f32(0.75 * fx["stale"][1])


def test_uniform_half_weight_is_dominated_by_pickconfigs_and_thief():
    """S:289 dominance: at w = 1/2 the uniform allocation is the thief's fair start, so
    fixed-config value <= PickConfigs(fair) <= thief (exact integer objectives)."""
    for cfg in (synth.CONFIG1, synth.CONFIG2):
        c = synth.SchedConfig(**{**cfg.__dict__, "n_inst": 200})
        inst = make_inst(c, 0, 200)
        fair = oracle.fair(inst)
        ts = oracle.thief(inst, oracle.STEEPEST)[2]
        tl = oracle.thief(inst, oracle.LITERAL)[2]
        for g in [oracle.HIGHEST_POST, 0] + list(range(1, inst.nG + 1)):
            a, cf, s, mean, bad = oracle.uniform(inst, g, 0.5)
            assert bad == 0
            for b in range(200):
                assert list(a[b]) == list(fair[b] if fair.ndim == 2 else fair)
                pc = oracle.pickconfigs(inst, b, fair)[0]
                assert int(s[b]) <= pc <= int(ts[b]) and pc <= int(tl[b])


def test_uniform_highest_post_ties_take_the_lowest_index():
    """U2 ("the configuration ... that results in the highest accuracy"): on a tie of the
    highest post-retraining accuracy the lowest-index config is the fixed one (C7's tie rule).
    Two configs of every stream are forced to share the maximum; the reported gamma (cfg bits
    0-4, 1-based) must be the lower of the two wherever a lambda is admissible."""
    c = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": 40})
    T = synth.sched_tables(c)
    post = (T["post"].numpy() * np.float32(0.5)).astype(np.float32)   # every real post < 1 ...
    cost = T["cost"].numpy()
    for b in range(40):
        for v in range(post.shape[1]):
            i, j = (3 + b + v) % 18, (11 + 2 * b + v) % 18
            lo_, hi_ = min(i, j), max(i, j)
            post[b, v, lo_] = post[b, v, hi_] = np.float32(1.0)   # ... but these two
    inst = oracle.Instances(T["stale"].numpy(), cost, post, T["lam_min_units"].numpy(),
                            T["lam_factor"].numpy(), c.units, c.steal_units, c.unit_gpu_seconds, c.a_min)
    a, cfg, s, mean, bad = oracle.uniform(inst)
    assert bad == 0
    checked = 0
    for b in range(40):
        for v in range(post.shape[1]):
            if (cfg[b, v] >> 5) == oracle.LAMBDA_NONE:
                continue
            i, j = (3 + b + v) % 18, (11 + 2 * b + v) % 18
            assert (cfg[b, v] & 31) == min(i, j) + 1
            checked += 1
    assert checked > 200


def test_uniform_weight_and_no_retraining():
    """U1: r_train = floor(share (1 - w)); fixed config 0 (no retraining) is stale x factor."""
    c = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": 20})
    inst = make_inst(c, 0, 20)
    for w in (0.1, 0.25, 0.9):
        a, cf, s, mean, bad = oracle.uniform(inst, 0, w)
        share = a[:, 0::2] + a[:, 1::2]
        assert (a.sum(1) == c.units).all()
        assert (a[:, 1::2] == np.floor(share * np.float32(1 - np.float32(w))).astype(int)).all()
        assert ((cf & 31) == 0).all()
        for b in range(20):
            tot = 0
            for v in range(c.n_streams):
                lam = cf[b, v] >> 5
                x = 0.0 if lam == 7 else f32(inst.lam_factor[b, v, lam]) * f32(inst.stale[b, v])
                tot += oracle.q32(f32(x))
            assert tot == int(s[b])


def test_pareto_spec_examples_and_properties():
    """singleton; equal accuracy, lower cost dominates; 20 random points = the
    dominance definition; the frontier is a staircase (cost ascending, accuracy strictly
    ascending) and every other point is dominated by a frontier point (Fig. 3 caption)."""
    assert int(oracle.pareto([[10.0]], [[0.9]])[0]) == 0b1
    assert int(oracle.pareto([[10.0, 5.0]], [[0.9, 0.9]])[0]) == 0b10
    rng = np.random.default_rng(31)
    for _ in range(300):
        n = int(rng.integers(1, 32))
        c = rng.choice([1.0, 2.0, 3.0, 5.0, 8.0], n).astype(np.float32) * rng.integers(1, 4, n)
        p = np.round(rng.uniform(0, 1, n), 1).astype(np.float32)
        c[rng.uniform(size=n) < 0.1] = np.inf                     # padding
        m = int(oracle.pareto(c[None], p[None])[0])
        on = [k for k in range(n) if m >> k & 1]
        for k in range(n):
            dom = any(j != k and np.isfinite(c[j]) and c[j] <= c[k] and p[j] >= p[k] and
                      (c[j] < c[k] or p[j] > p[k]) for j in range(n))
            assert (k in on) == (np.isfinite(c[k]) and not dom)
        pts = sorted(set((float(c[k]), float(p[k])) for k in on))
        for (c0, p0), (c1, p1) in zip(pts, pts[1:]):
            assert c0 < c1 and p0 < p1
        for k in range(n):
            if np.isfinite(c[k]) and k not in on:
                assert any(c[j] <= c[k] and p[j] >= p[k] for j in on)


def test_pareto_invalid_data_and_empty_input():
    """R-ERR for the frontier: a NaN, negative or -INF cost, or a real config's accuracy
    outside [0, 1] (or NaN) invalidates the set (mask 0, counted); +INF is padding and its
    accuracy is ignored; S:115's empty input (no configurations) is an argument error."""
    inf, nan = float("inf"), float("nan")
    c = np.array([[1.0, 2.0], [nan, 2.0], [-1.0, 2.0], [-inf, 2.0], [1.0, 2.0], [1.0, 2.0], [1.0, inf]],
                 np.float32)
    p = np.array([[0.5, 0.6], [0.5, 0.6], [0.5, 0.6], [0.5, 0.6], [1.5, 0.6], [nan, 0.6], [0.5, 7.0]],
                 np.float32)
    m, bad = oracle.pareto(c, p, with_bad=True)
    assert bad == 5
    assert m.tolist() == [0b11, 0, 0, 0, 0, 0, 0b01]
    with pytest.raises(ValueError):
        oracle.pareto(np.zeros((3, 0), np.float32), np.zeros((3, 0), np.float32))


def test_prune_reading_vs_spec_example():
    """PN1 measures distance from the Pareto boundary VERTICALLY (accuracy gap at the config's
    cost), not as SPEC.md's relative cost distance.  P:1179-1180 fixes neither
    ("significantly distant from the configurations on the Pareto curve").  Consequence,
    pinned: SPEC's example (a config matched in accuracy by one 10x cheaper in every
    window, margin 0.5) is KEPT here -- its accuracy gap is 0 -- while a config whose accuracy
    falls below the boundary by more than the margin in most windows is dropped whatever its
    cost ratio."""
    c = np.array([[1.0, 10.0]], np.float32)
    A = np.array([[[.6, .6], [.7, .7], [.5, .5]]], np.float32)
    assert int(oracle.prune(c, A, 0.5)[0][0]) == 0b11     # S:132's drop is not this reading's
    A2 = np.array([[[.6, .4], [.7, .5], [.5, .3]]], np.float32)
    assert int(oracle.prune(c, A2, 0.15)[0][0]) == 0b01   # gap .2 > .15 in 3/3 windows
    assert int(oracle.prune(c, A2, 0.25)[0][0]) == 0b11   # gap .2 <= .25: kept
    # a costlier config ABOVE the cheaper one's accuracy is on the boundary: gap 0
    A3 = np.array([[[.5, .9], [.5, .9], [.5, .9]]], np.float32)
    assert int(oracle.prune(c, A3, 0.0)[0][0]) == 0b11


def test_prune_worked_examples():
    """PN1-PN3 on hand-worked cases: costs 1, 2, 3 and three windows.
    w0 = (.5, .7, .6): config 2 sits .1 below the boundary (.7 at cost <= 3); w1 = (.6,
    .62, .64): on the boundary everywhere; w2 = (.7, .6, .5): configs 1, 2 are .1 and .2
    below.  Margin .05: config 1 far in 1/3 windows (kept), config 2 in 2/3 (pruned)."""
    nan = float("nan")
    c = np.array([[1.0, 2.0, 3.0]], np.float32)
    A = np.array([[[.5, .7, .6], [.6, .62, .64], [.7, .6, .5]]], np.float32)
    assert oracle.prune(c, A, 0.05) == (np.array([0b011], np.uint32), 0)
    # exactly half of the measured windows far: kept ("usually" = strict majority)
    assert int(oracle.prune(c, A[:, :2], 0.05)[0][0]) == 0b111
    # unmeasured windows do not count: config 2 measured in w0 only, far there
    A2 = A[:, :2].copy()
    A2[0, 1, 2] = nan
    assert int(oracle.prune(c, A2, 0.05)[0][0]) == 0b011
    # never measured: kept; a margin above every gap keeps all, a negative one prunes
    # every measured config
    A3 = A.copy()
    A3[0, :, 2] = nan
    assert int(oracle.prune(c, A3, 0.05)[0][0]) == 0b111
    assert int(oracle.prune(c, A, 1.0)[0][0]) == 0b111
    assert int(oracle.prune(c, A, -1.0)[0][0]) == 0
    assert int(oracle.prune(c, A3, -1.0)[0][0]) == 0b100
    # padding (cost +INF) is never kept and does not raise the boundary
    cp = np.array([[1.0, 2.0, np.inf]], np.float32)
    Ap = np.array([[[.5, .6, 1.0]]], np.float32)
    assert int(oracle.prune(cp, Ap, 0.0)[0][0]) == 0b011
    # equal cost counts as "not above": the worse of two equal-cost configs is far
    assert int(oracle.prune(np.array([[1.0, 1.0]], np.float32),
                            np.array([[[.5, .6]]], np.float32), 0.05)[0][0]) == 0b10
    # invalid data: mask 0 and counted; a padding config's accuracy is not data
    bad_c = np.array([[1.0, nan, 3.0]], np.float32)
    assert oracle.prune(bad_c, A, 0.05) == (np.array([0], np.uint32), 1)
    Ab = A.copy()
    Ab[0, 1, 0] = 1.5
    assert oracle.prune(c, Ab, 0.05) == (np.array([0], np.uint32), 1)
    Apb = Ap.copy()
    Apb[0, 0, 2] = 7.0
    assert oracle.prune(cp, Apb, 0.0)[1] == 0


def test_prune_invariants_and_pareto_relation():
    """Random tie-heavy sets: the mask permutes with the configs, ignores the window order,
    grows with the margin; with one window, margin 0 and acc = post it keeps the Pareto
    frontier (PR1, pinned above) plus exactly the configs whose accuracy some real config
    at no higher cost matches."""
    rng = np.random.default_rng(41)
    for _ in range(200):
        n = int(rng.integers(1, 32))
        H = int(rng.integers(0, 7))
        c = (rng.choice([1.0, 2.0, 3.0, 5.0], n) * rng.integers(1, 3, n)).astype(np.float32)
        c[rng.uniform(size=n) < 0.1] = np.inf
        A = np.round(rng.uniform(0, 1, (H, n)), 1).astype(np.float32)
        A[rng.uniform(size=(H, n)) < 0.2] = np.nan
        m = float(rng.choice([0.0, 0.1, 0.25]))
        keep = int(oracle.prune(c[None], A[None], m)[0][0])
        perm = rng.permutation(n)
        kp = int(oracle.prune(c[perm][None], A[:, perm][None], m)[0][0])
        assert kp == sum(1 << i for i in range(n) if keep >> int(perm[i]) & 1)
        assert int(oracle.prune(c[None], A[rng.permutation(H)][None], m)[0][0]) == keep
        assert keep & ~int(oracle.prune(c[None], A[None], m + 0.2)[0][0]) == 0
        p = np.round(rng.uniform(0, 1, n), 1).astype(np.float32)
        k1 = int(oracle.prune(c[None], p[None, None], 0.0)[0][0])
        par = int(oracle.pareto(c[None], p[None])[0])
        assert par & ~k1 == 0
        for k in range(n):
            if k1 >> k & 1 and not par >> k & 1:
                assert any(j != k and np.isfinite(c[j]) and c[j] <= c[k] and p[j] == p[k] for j in range(n))
            if np.isfinite(c[k]) and not k1 >> k & 1:
                assert any(np.isfinite(c[j]) and c[j] <= c[k] and p[j] > p[k] for j in range(n))


# ---------------------------------------------------------------------------
# NEXT-2: micro-profiler curve fit
# ---------------------------------------------------------------------------
def _curve(b0, b1, b2, k):
    return 1.0 - (1.0 / (b0 * k + b1) + b2)


def test_curve_fit_spec_examples():
    """S:155 constant data -> constant fit; S:156 noiseless round trip within 1e-3 at k = 30;
    S:161 the (0.5, 1.0, 0.1) curve at 30 epochs is 0.8375."""
    k = np.arange(1, 6, dtype=np.float64)
    a = np.stack([np.full(5, 0.7), _curve(0.5, 1.0, 0.1, k)]).astype(np.float32)
    for K in (1, 5, 30, 100):
        pred, prm, bad = oracle.curve_fit(a, np.array([K, K]))
        assert bad == 0
        assert pred[0] == pytest.approx(0.7, abs=1e-6)
        assert pred[1] == pytest.approx(_curve(0.5, 1.0, 0.1, K), abs=1e-3)
    assert _curve(0.5, 1.0, 0.1, 30) == pytest.approx(0.8375)


def test_curve_fit_noisy_median_error():
    """sigma = 0.02 noise on k = 1..5, median absolute error at k = 30 over 200 random
    curves of the family < 0.058 (the paper's 5.8% median error)."""
    rng = np.random.default_rng(51)
    k = np.arange(1, 6, dtype=np.float64)
    b0, b1, b2 = rng.uniform(0.2, 2.0, 200), rng.uniform(0.8, 3.0, 200), rng.uniform(0.0, 0.3, 200)
    a = np.clip(_curve(b0[:, None], b1[:, None], b2[:, None], k) + rng.normal(0, 0.02, (200, 5)), 0, 1)
    pred, _, bad = oracle.curve_fit(a.astype(np.float32), np.full(200, 30))
    assert bad == 0
    assert np.median(np.abs(pred - _curve(b0, b1, b2, 30))) < 0.058


def test_curve_fit_nnls_and_grid_optimal():
    """CF1-CF2 against an independent solver: for every grid c the fp64 active-set-free NNLS
    (scipy.optimize.nnls) optimum is no better than the chosen c's by more than rounding;
    alpha, beta2 >= 0; the extrapolation is non-decreasing in the epoch count."""
    from scipy.optimize import nnls
    rng = np.random.default_rng(52)
    S = 60
    a = np.clip(rng.uniform(0.3, 0.9, (S, 1)) + np.cumsum(rng.uniform(-0.03, 0.08, (S, 5)), 1), 0, 1)
    a = a.astype(np.float32)
    pred, prm, bad = oracle.curve_fit(a, np.full(S, 30))
    assert bad == 0 and (prm[:, 0] >= 0).all() and (prm[:, 2] >= 0).all()
    y = 1.0 - a.astype(np.float64)
    for s in range(S):
        def sse(c):
            X = np.stack([1.0 / (np.arange(1, 6) + c), np.ones(5)], 1)
            return nnls(X, y[s])[1] ** 2
        chosen = sse(float(prm[s, 1]))
        best = min(sse(i / 8) for i in range(257))
        assert chosen <= best + 1e-6
        p2, _, _ = oracle.curve_fit(a[s:s + 1], np.array([60]))
        assert p2[0] >= pred[s] - 1e-7


def test_curve_fit_grid_ties_and_clamp():
    """CF2: constant accuracy is fitted exactly (alpha = 0, beta2 = 1 - acc) at EVERY grid c --
    the SSE is 0 throughout -- so the lowest grid index, c = 0, is the one reported.  CF3: the
    extrapolation is clamped to [0, 1]; accuracies that start at 0 and barely rise give fits
    whose value at epoch 1 lies below 0 (found by search; checked here from the returned
    parameters), and the prediction is 0, never negative."""
    for n in (2, 5):
        pred, prm, bad = oracle.curve_fit(np.full((1, n), 0.5, np.float32), np.array([7]))
        assert bad == 0 and prm[0].tolist() == [0.0, 0.0, 0.5] and pred[0] == 0.5
    cases = np.array([[0.0, 1 / 64, 6 / 64, 6 / 64], [0.0, 0.0, 3 / 64, 6 / 64]], np.float32)
    pred, prm, bad = oracle.curve_fit(cases, np.array([1, 1]))
    assert bad == 0
    for i in range(2):
        al, c, b2 = (float(x) for x in prm[i])
        assert 1.0 - (al / (1.0 + c) + b2) < -1e-3      # the unclamped model value
        assert pred[i] == 0.0


def test_curve_fit_invalid():
    a = np.array([[0.5, 0.6, 1.2, 0.7, 0.8], [0.5, 0.6, 0.7, 0.7, 0.8]], np.float32)
    pred, _, bad = oracle.curve_fit(a, np.array([30, 0]))
    assert bad == 2 and (pred == 0).all()


# ---------------------------------------------------------------------------
# NEXT-1: the window as a timeline, thief re-invoked at each completion
# ---------------------------------------------------------------------------
def test_window_single_stream_closed_form():
    """One stream, U = 4, uT = 10 GPU-s/unit, stale 0.5, one config (cost 10, post 0.9), one
    lambda (factor 1).  The thief ends at r_train = 3 (window average 0.9 - 0.4/3 beats
    r_train = 2's 0.7 and r_train = 1's 0.5), so retraining ends at tau = 1/3; re-invoked,
    the stream is done (model 0.9).  Realized average = tau1 0.5 + (1 - tau1) 0.9, written
    out in binary32 (W4-W6), and 23/30 in exact rationals."""
    inst = oracle.Instances([[0.5]], [[[10.0]]], [[[0.9]]], [[[1]]], [[[1.0]]], 4, 1, 10.0, 0.0)
    a, c, s, mean, steps, _ = oracle.thief(inst, oracle.STEEPEST)
    assert a.tolist() == [[1, 3]]
    avg, ev, done, bad = oracle.window(inst, oracle.STEEPEST)
    f = np.float32(10.0) / (np.float32(3.0) * np.float32(10.0))
    t1 = np.float32(0.0) + f * (np.float32(1.0) - np.float32(0.0))
    seg1 = t1 * (np.float32(1.0) * np.float32(0.5))
    seg2 = (np.float32(1.0) - t1) * (np.float32(1.0) * np.float32(0.9))
    assert bad == 0 and ev[0] == 2 and done[0, 0] == t1
    assert avg[0] == np.float32(np.float32(0.0) + seg1 + seg2) / np.float32(1.0)
    assert avg[0] == pytest.approx(23 / 30, abs=1e-6)


def test_window_partial_progress_two_streams():
    """W3 (retraining branch) and W6 on a hand-worked two-stream timeline.

    U = 4, steal_units 8 > every share, so no steal is ever possible (C14) and every
    invocation keeps the fair start (C9): r_infer = r_train = 1 per stream.  uT = 10, one
    lambda (factor 1, needs 1 unit), a_MIN 0, stale 0.5.
      A: cost 2.5, post 0.75 -> f = 1/4, window value 0.6875 > 0.5: retrains, done at 1/4.
      B: cost 7.5, post 0.75 -> f = 3/4, value 0.5625 > 0.5: retrains, done at 3/4.
    Invocation 1 (tau = 0) ends at tau* = 1/4 (W4).  B has done (1/4)/(3/4) = 1/3 of its
    work, so R_B = 7.5 (1 - 1/3) = 5 (W6).  Invocation 2 (tau = 1/4): B's residual cost is
    R_B / (1 - 1/4) = 20/3 (W3), f = 2/3, so B completes at 1/4 + (2/3)(3/4) = 3/4 -- the
    progress carried over exactly.  Invocation 3 at 3/4: both done, run to 1.
    Realized averages (W5): A = 1/4 * 0.5 + 3/4 * 0.75 = 0.6875,
    B = 3/4 * 0.5 + 1/4 * 0.75 = 0.5625; window average 0.625; 3 invocations.
    Dropping the residual rescale (B done at 5/8) or keeping the done fraction instead of
    the remaining one (B done at 1/2) both move B's completion time."""
    inst = oracle.Instances([[0.5, 0.5]], [[[2.5], [7.5]]], [[[0.75], [0.75]]], [[[1], [1]]],
                            [[[1.0], [1.0]]], 4, 8, 10.0, 0.0)
    a, c, _, _, steps, _ = oracle.thief(inst, oracle.STEEPEST)
    assert a.tolist() == [[1, 1, 1, 1]] and steps[0] == 0 and (c & 31).tolist() == [[1, 1]]
    for mode in (oracle.STEEPEST, oracle.LITERAL):
        avg, ev, done, bad = oracle.window(inst, mode)
        assert bad == 0 and ev[0] == 3
        assert done[0, 0] == np.float32(0.25)
        assert done[0, 1] == pytest.approx(0.75, abs=1e-6)
        exact_A = Fr(1, 4) * Fr(1, 2) + Fr(3, 4) * Fr(3, 4)
        exact_B = Fr(3, 4) * Fr(1, 2) + Fr(1, 4) * Fr(3, 4)
        assert exact_A == Fr(11, 16) and exact_B == Fr(9, 16)
        assert avg[0] == pytest.approx(float((exact_A + exact_B) / 2), abs=2e-6)


def test_window_idle_stream_starts_after_a_completion():
    """W3 (idle branch) on a hand-worked two-stream timeline: units freed by a finished
    retraining let an idle stream start, with its cost scaled to the shorter residual window.

    U = 4, steal_units 1, uT = 10, one lambda (factor 1, needs 1 unit), a_MIN 0, stale 0.5.
      A: cost 5, post 0.75: f(1) = 1/2 (value 0.625), f(2) = 1/4 (value 0.6875).
      B: cost 12, post 0.875: f(1) = 6/5 > 1 (infeasible), f(2) = 3/5 (value 0.65).
    tau = 0, fair start (1, 1 | 1, 1): the only improving steal moves B's training unit to
    A's (+1/16; giving A's to B is +0.025 - 0.125 < 0; any inference steal zeroes a
    stream), after which nothing improves, in both modes: A (1, 2) done at 1/4, B (1, 0)
    idle.  tau = 1/4: A's training unit is worthless to A (done), and B's residual cost
    is 12 / (3/4) = 16 (W3), so with 2 units f = 16/20 = 4/5 (value 0.575 > 0.5): B
    starts and completes at 1/4 + (4/5)(3/4) = 17/20.  Realized (W5):
    A = 1/4 * 0.5 + 3/4 * 0.75 = 0.6875,
    B = 1/4 * 0.5 + (3/5) * 0.5 + (3/20) * 0.875 = 0.55625, average 0.621875.
    Without the rescale B would finish at 1/4 + (3/5)(3/4) = 7/10."""
    inst = oracle.Instances([[0.5, 0.5]], [[[5.0], [12.0]]], [[[0.75], [0.875]]], [[[1], [1]]],
                            [[[1.0], [1.0]]], 4, 1, 10.0, 0.0)
    for mode in (oracle.STEEPEST, oracle.LITERAL):
        a, c, _, _, steps, _ = oracle.thief(inst, mode)
        assert a.tolist() == [[1, 2, 1, 0]] and (c & 31).tolist() == [[1, 0]]
        avg, ev, done, bad = oracle.window(inst, mode)
        assert bad == 0 and ev[0] == 3
        assert done[0, 0] == np.float32(0.25)
        assert done[0, 1] == pytest.approx(17 / 20, abs=1e-6)
        exact_A = Fr(1, 4) * Fr(1, 2) + Fr(3, 4) * Fr(3, 4)
        exact_B = Fr(1, 4) * Fr(1, 2) + Fr(3, 5) * Fr(1, 2) + Fr(3, 20) * Fr(7, 8)
        assert avg[0] == pytest.approx(float((exact_A + exact_B) / 2), abs=2e-6)
        assert float((exact_A + exact_B) / 2) == 0.621875


def test_window_without_retraining_is_the_thief_estimate():
    """No retraining config finishes (all +inf): one invocation over the whole window and
    the realized average equals the thief's estimate (W5 with tau* = 1)."""
    c = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": 50})
    inst = make_inst(c, 0, 50)
    inst2 = oracle.Instances(inst.stale, np.full_like(inst.cost, np.inf), inst.post, inst.lam_min_units,
                             inst.lam_factor, inst.units, inst.steal_units, inst.unit_gpu_seconds, inst.a_min)
    avg, ev, done, bad = oracle.window(inst2, oracle.STEEPEST)
    mean = oracle.thief(inst2, oracle.STEEPEST)[3]
    assert bad == 0 and (ev == 1).all() and (done == 1).all()
    np.testing.assert_allclose(avg, mean, atol=2e-6)


def test_window_invariants():
    """At most V + 1 invocations; every completion time in (0, 1]; a stream completes at most
    once; 0 <= average <= 1; both modes; re-invocation (freed units return to inference,
    C4(b)) does not lose to the t = 0 estimate on average over many instances."""
    for cfg in (synth.CONFIG1, synth.CONFIG2):
        c = synth.SchedConfig(**{**cfg.__dict__, "n_inst": 120})
        inst = make_inst(c, 0, 120)
        for mode in (oracle.STEEPEST, oracle.LITERAL):
            avg, ev, done, bad = oracle.window(inst, mode)
            assert bad == 0
            assert (ev >= 1).all() and (ev <= inst.V + 1).all()
            assert ((done > 0) & (done <= 1)).all()
            assert ((avg >= 0) & (avg <= 1)).all()
            assert avg.mean() >= oracle.thief(inst, mode)[3].mean() - 1e-3
