"""CPU oracle for Ekya's scheduling hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2012_10557_b200`` never imports it, and this package never imports the
product (they share no code; the only common dependency is the seeded input
generator ``synth``, which holds none of the method's arithmetic).

The arithmetic lives in plain C (``ekya_oracle.c``, one fp32 rounding per
operation, ``-ffp-contract=off``); this module is ctypes marshalling of numpy
arrays plus the gcc build step.  Function-by-function citations are in the C
file; the readings of the paper it follows are DESIGN.md section 3.

Parity status: every function is pinned by ``tests/test_oracle_pins.py`` except
the two thief readings, whose *trajectories* the paper never prints; they are
pinned by a line-by-line transliteration of Algorithm 1 plus invariants
(DESIGN.md section 4 lists what pins each function).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ekya_oracle.c")
_LIB = os.path.join(_HERE, "_build", "libekya_oracle.so")

LAMBDA_NONE = 7
LMU_PAD = 0xFFFF
STEEPEST = 0
LITERAL = 1
RADIUS = 0
CLUSTER = 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2, no FMA contraction, no fast-math."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fno-math-errno",
           "-fPIC", "-shared", "-Wall", "-Wextra", "-o", _LIB, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB


class Dims(ctypes.Structure):
    _fields_ = [("n_inst", ctypes.c_int32), ("n_streams", ctypes.c_int32),
                ("n_gamma", ctypes.c_int32), ("n_lambda", ctypes.c_int32),
                ("units", ctypes.c_int32), ("steal_units", ctypes.c_int32),
                ("unit_gpu_seconds", ctypes.c_float), ("a_min", ctypes.c_float)]


class ProfileDims(ctypes.Structure):
    _fields_ = [("n_query", ctypes.c_int32), ("n_hist", ctypes.c_int32),
                ("n_class", ctypes.c_int32), ("n_gamma", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("tau", ctypes.c_float),
                ("k", ctypes.c_int32), ("max_iter", ctypes.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        L = _lib
        L.orc_retrain_fraction.restype = ctypes.c_float
        L.orc_retrain_fraction.argtypes = [ctypes.c_float, ctypes.c_int32, ctypes.c_float]
        L.orc_gamma_feasible.restype = ctypes.c_int32
        L.orc_gamma_feasible.argtypes = [ctypes.c_float, ctypes.c_int32, ctypes.c_float]
        L.orc_window_accuracy.restype = ctypes.c_float
        L.orc_window_accuracy.argtypes = [ctypes.c_float] * 3 + [ctypes.c_int32, ctypes.c_float]
        L.orc_q32.restype = ctypes.c_uint64
        L.orc_q32.argtypes = [ctypes.c_float]
        L.orc_stream_value.restype = ctypes.c_float
        L.orc_stream_value.argtypes = [ctypes.POINTER(Dims), ctypes.c_float, P, P, P, P,
                                       ctypes.c_int32, ctypes.c_int32, P]
        L.orc_pickconfigs.restype = ctypes.c_uint64
        L.orc_pickconfigs.argtypes = [ctypes.POINTER(Dims), ctypes.c_int64, P, P, P, P, P, P, P, P]
        L.orc_fair.restype = None
        L.orc_fair.argtypes = [ctypes.POINTER(Dims), P]
        L.orc_eval_grid.restype = ctypes.c_int64
        L.orc_eval_grid.argtypes = [ctypes.POINTER(Dims), P, P, P, P, P, P, P]
        L.orc_eval_list.restype = ctypes.c_int64
        L.orc_eval_list.argtypes = [ctypes.POINTER(Dims), P, P, P, P, P, ctypes.c_int32, P, P, P, P]
        L.orc_thief.restype = ctypes.c_int64
        L.orc_thief.argtypes = [ctypes.POINTER(Dims), P, P, P, P, P, ctypes.c_int32, P, P, P, P, P]
        L.orc_bruteforce.restype = ctypes.c_int64
        L.orc_bruteforce.argtypes = [ctypes.POINTER(Dims), P, P, P, P, P, P, P, P]
        L.orc_profile.restype = ctypes.c_int64
        L.orc_profile.argtypes = [ctypes.POINTER(ProfileDims), P, P, P, P, P, P, P]
        L.orc_profile_ex.restype = ctypes.c_int64
        L.orc_profile_ex.argtypes = [ctypes.POINTER(ProfileDims), P, P, P, P, P, P, P, P]
        L.orc_quantize_frac.argtypes = [ctypes.c_int64, ctypes.c_int32]
        L.orc_quantize_frac.restype = ctypes.c_int32
        L.orc_uniform.argtypes = [ctypes.POINTER(Dims), P, P, P, P, P, ctypes.c_int32, ctypes.c_float, P, P, P, P]
        L.orc_uniform.restype = ctypes.c_int64
        L.orc_pareto.argtypes = [ctypes.c_int64, ctypes.c_int32, P, P, P]
        L.orc_pareto.restype = ctypes.c_int64
        L.orc_prune.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, ctypes.c_float, P]
        L.orc_prune.restype = ctypes.c_int64
        L.orc_window.argtypes = [ctypes.POINTER(Dims), P, P, P, P, P, ctypes.c_int32, P, P, P]
        L.orc_window.restype = ctypes.c_int64
        L.orc_curve_fit.argtypes = [ctypes.c_int64, ctypes.c_int32, P, P, P, P]
        L.orc_curve_fit.restype = ctypes.c_int64
        L.orc_pack.argtypes = [ctypes.c_int32, P, ctypes.c_int32, P, P]
        L.orc_pack.restype = ctypes.c_int64
        L.orc_place.argtypes = [ctypes.c_int32] * 4 + [P] * 6
        L.orc_place.restype = ctypes.c_int64
        L.orc_checkpoint.argtypes = [ctypes.c_int64] + [P] * 8
        L.orc_checkpoint.restype = ctypes.c_int64
    return _lib


# ---------------------------------------------------------------------------
# marshalling helpers
# ---------------------------------------------------------------------------
def _c(a, dtype):
    a = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Instances:
    """Host-side batch of scheduling instances (numpy, instance-major SoA).

    stale [B,V] f32; cost, post [B,V,nG] f32; lam_min_units [B,V,nL] u16;
    lam_factor [B,V,nL] f32; scalars units, steal_units, unit_gpu_seconds, a_min.
    """

    def __init__(self, stale, cost, post, lam_min_units, lam_factor, units, steal_units,
                 unit_gpu_seconds, a_min):
        self.stale = _c(stale, np.float32)
        B, V = self.stale.shape

        def shaped(a, dt):
            a = _c(a, dt)
            return a if a.ndim == 3 else a.reshape(B, V, -1)
        self.cost = shaped(cost, np.float32)
        self.post = shaped(post, np.float32)
        self.lam_min_units = shaped(lam_min_units, np.uint16)
        self.lam_factor = shaped(lam_factor, np.float32)
        self.units = int(units)
        self.steal_units = int(steal_units)
        self.unit_gpu_seconds = float(unit_gpu_seconds)
        self.a_min = float(a_min)

    @property
    def B(self):
        return self.stale.shape[0]

    @property
    def V(self):
        return self.stale.shape[1]

    @property
    def nG(self):
        return self.cost.shape[2]

    @property
    def nL(self):
        return self.lam_factor.shape[2]

    def dims(self):
        return Dims(self.B, self.V, self.nG, self.nL, self.units, self.steal_units,
                    self.unit_gpu_seconds, self.a_min)

    def tables(self):
        return (_p(self.stale), _p(self.cost), _p(self.post), _p(self.lam_min_units),
                _p(self.lam_factor))

    def subset(self, idx):
        idx = np.asarray(idx)
        return Instances(self.stale[idx], self.cost[idx], self.post[idx], self.lam_min_units[idx],
                         self.lam_factor[idx], self.units, self.steal_units,
                         self.unit_gpu_seconds, self.a_min)


def n_cells(units: int) -> int:
    return (units + 1) * (units + 2) // 2


# ---------------------------------------------------------------------------
# primitives
# ---------------------------------------------------------------------------
def retrain_fraction(cost, rt, uT):
    return lib().orc_retrain_fraction(cost, rt, uT)


def gamma_feasible(cost, rt, uT):
    return bool(lib().orc_gamma_feasible(cost, rt, uT))


def window_accuracy(stale, post, cost, rt, uT):
    return lib().orc_window_accuracy(stale, post, cost, rt, uT)


def q32(x):
    return int(lib().orc_q32(x))


def stream_value(inst: Instances, b: int, v: int, rt: int, ri: int):
    d = inst.dims()
    cfg = np.zeros(1, np.uint8)
    cost = np.ascontiguousarray(inst.cost[b, v])
    post = np.ascontiguousarray(inst.post[b, v])
    lmu = np.ascontiguousarray(inst.lam_min_units[b, v])
    lf = np.ascontiguousarray(inst.lam_factor[b, v])
    val = lib().orc_stream_value(ctypes.byref(d), float(inst.stale[b, v]), _p(cost), _p(post),
                                 _p(lmu), _p(lf), rt, ri, _p(cfg))
    return float(np.float32(val)), int(cfg[0])


def pickconfigs(inst: Instances, b: int, alloc):
    d = inst.dims()
    a = _c(alloc, np.int32)
    cfg = np.zeros(inst.V, np.uint8)
    vals = np.zeros(inst.V, np.float32)
    s = lib().orc_pickconfigs(ctypes.byref(d), b, *inst.tables(), _p(a), _p(cfg), _p(vals))
    return int(s), cfg, vals


def fair(inst: Instances):
    d = inst.dims()
    a = np.zeros(2 * inst.V, np.int32)
    lib().orc_fair(ctypes.byref(d), _p(a))
    return a


def mean_from_q32(s, V):
    return np.float32(np.float64(s) / (np.float64(V) * 4294967296.0))


# ---------------------------------------------------------------------------
# batched procedures
# ---------------------------------------------------------------------------
def eval_grid(inst: Instances):
    d = inst.dims()
    nc = n_cells(inst.units)
    grid = np.zeros((inst.B, inst.V, nc), np.float32)
    cfg = np.zeros((inst.B, inst.V, nc), np.uint8)
    bad = lib().orc_eval_grid(ctypes.byref(d), *inst.tables(), _p(grid), _p(cfg))
    if bad < 0:
        raise ValueError("oracle: invalid dims")
    return grid, cfg, int(bad)


def eval_list(inst: Instances, alloc):
    d = inst.dims()
    alloc = _c(alloc, np.uint16)
    n = alloc.shape[1]
    s = np.zeros((inst.B, n), np.uint64)
    mean = np.zeros((inst.B, n), np.float32)
    cfg = np.zeros((inst.B, n, inst.V), np.uint8)
    bad = lib().orc_eval_list(ctypes.byref(d), *inst.tables(), n, _p(alloc), _p(s), _p(mean),
                              _p(cfg))
    if bad < 0:
        raise ValueError("oracle: invalid dims")
    return s, mean, cfg, int(bad)


def thief(inst: Instances, mode: int = STEEPEST):
    d = inst.dims()
    B, V = inst.B, inst.V
    alloc = np.zeros((B, 2 * V), np.uint16)
    cfg = np.zeros((B, V), np.uint8)
    s = np.zeros(B, np.uint64)
    mean = np.zeros(B, np.float32)
    steps = np.zeros(B, np.uint32)
    bad = lib().orc_thief(ctypes.byref(d), *inst.tables(), mode, _p(alloc), _p(cfg), _p(s),
                          _p(mean), _p(steps))
    if bad < 0:
        raise ValueError("oracle: invalid dims/mode")
    return alloc, cfg, s, mean, steps, int(bad)


def host_threads() -> int:
    """Host cores this process may use (the oracle's thread pool size)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def per_instance_parallel(fn, inst: Instances, *args, threads: int | None = None):
    """Run fn(inst_subset, *args) over instance blocks on a thread pool of all host cores and
    concatenate the array outputs (trailing int = bad count, summed).  Array arguments whose
    first dimension is the instance count (e.g. LIST rows [B][N][J]) are sliced with the
    block.  Marshalling only: the instances are independent and each block runs the
    unchanged single-threaded oracle code; ctypes releases the GIL inside the C call."""
    from concurrent.futures import ThreadPoolExecutor
    threads = threads or host_threads()
    B = inst.B
    if B == 0 or threads <= 1:
        return fn(inst, *args)
    bounds = np.linspace(0, B, min(B, threads * 4) + 1).astype(np.int64)
    blocks = [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1) if bounds[i + 1] > bounds[i]]
    lib()   # load once before the threads start

    def block(lh):
        idx = np.arange(lh[0], lh[1])
        a = [x[lh[0]:lh[1]] if isinstance(x, np.ndarray) and x.ndim >= 1 and x.shape[0] == B else x
             for x in args]
        return fn(inst.subset(idx), *a)
    with ThreadPoolExecutor(max_workers=threads) as ex:
        parts = list(ex.map(block, blocks))
    out = []
    for i, first in enumerate(parts[0]):
        if isinstance(first, np.ndarray):
            out.append(np.concatenate([p[i] for p in parts]))
        else:
            out.append(sum(p[i] for p in parts))
    return tuple(out)


def bruteforce(inst: Instances):
    d = inst.dims()
    B, V = inst.B, inst.V
    alloc = np.zeros((B, 2 * V), np.uint16)
    cfg = np.zeros((B, V), np.uint8)
    s = np.zeros(B, np.uint64)
    bad = lib().orc_bruteforce(ctypes.byref(d), *inst.tables(), _p(alloc), _p(cfg), _p(s))
    if bad == -2:
        raise ValueError("oracle: instance too large for brute force")
    if bad < 0:
        raise ValueError("oracle: invalid dims")
    return alloc, cfg, s, int(bad)


def profile(cur, hist, hist_acc, fallback, mode=RADIUS, tau=0.2, k=5, max_iter=100, with_passes=False):
    """A1 estimates: (est [Q][G], n [Q][G], cluster [Q][H+1] or None, bad), and with
    with_passes the Lloyd assignment passes per query [Q] (telemetry) appended."""
    cur = _c(cur, np.float32)
    Q, C = cur.shape
    fallback = _c(fallback, np.float32)
    G = fallback.shape[-1]
    fallback = fallback.reshape(Q, G)
    hist = _c(hist, np.float32)
    H = hist.shape[1] if hist.ndim == 3 else hist.size // max(1, Q * C)
    hist = hist.reshape(Q, H, C)
    hist_acc = _c(hist_acc, np.float32).reshape(Q, H, G)
    pd = ProfileDims(Q, H, C, G, mode, tau, k, max_iter)
    est = np.zeros((Q, G), np.float32)
    n = np.zeros((Q, G), np.int32)
    cl = np.zeros((Q, H + 1), np.int32)
    passes = np.zeros(Q, np.int32)
    bad = lib().orc_profile_ex(ctypes.byref(pd), _p(cur), _p(hist), _p(hist_acc), _p(fallback),
                               _p(est), _p(n), _p(cl), _p(passes))
    if bad < 0:
        raise ValueError("oracle: invalid profile dims")
    out = (est, n, (cl if mode == CLUSTER else None), int(bad))
    return out + (passes,) if with_passes else out


Q_ONE = 65536   # one GPU in quanta of 2^-16 GPU (placement outputs)


def quantize_frac(r: int, units: int) -> int:
    """PL1: fractional GPU share r/U quantized down to 2^-k, in 2^-16 quanta."""
    return int(lib().orc_quantize_frac(int(r), int(units)))


def pack(q, gpus: int):
    """S:333-339 first-fit decreasing of demands q (2^-16 GPU quanta); returns (gpu per job, load)."""
    q = _c(q, np.uint32).reshape(-1)
    g = np.zeros(q.size, np.int16)
    load = np.zeros(gpus, np.uint32)
    lib().orc_pack(q.size, _p(q), gpus, _p(g), _p(load))
    return g, load


def place(alloc, units: int, gpus: int):
    """Placement onto GPUs (readings PL1-PL3).  alloc [B][J] u16.
    Returns piece_job [B][J+G] u16, piece_q [B][J+G] u32, piece_gpu [B][J+G] i16,
    n_pieces [B] u16, gpu_load [B][G] u32, bad."""
    alloc = _c(alloc, np.uint16)
    B, J = alloc.shape
    P = J + gpus
    pj = np.zeros((B, P), np.uint16)
    pq = np.zeros((B, P), np.uint32)
    pg = np.zeros((B, P), np.int16)
    npc = np.zeros(B, np.uint16)
    load = np.zeros((B, gpus), np.uint32)
    bad = lib().orc_place(B, J, units, gpus, _p(alloc), _p(pj), _p(pq), _p(pg), _p(npc), _p(load))
    if bad < 0:
        raise ValueError("oracle: invalid placement dims")
    return pj, pq, pg, npc, load, int(bad)


def checkpoint(tau, t, T, a, a_star, A, delta_ckpt):
    """Checkpoint decision (draft P:62-81, reading CK1): (tau-t)(a*-a) > delta A."""
    arrs = [_c(x, np.float32).reshape(-1) for x in (tau, t, T, a, a_star, A, delta_ckpt)]
    out = np.zeros(arrs[0].size, np.uint8)
    bad = lib().orc_checkpoint(arrs[0].size, *(_p(x) for x in arrs), _p(out))
    return out, int(bad)


HIGHEST_POST = -1   # uniform baseline: each stream's highest-accuracy config


def uniform(inst: Instances, fixed_gamma: int = HIGHEST_POST, inference_weight: float = 0.5):
    """Uniform baseline (readings U1, U2): alloc, cfg, sum, mean, bad."""
    d = inst.dims()
    B, V = inst.B, inst.V
    alloc = np.zeros((B, 2 * V), np.uint16)
    cfg = np.zeros((B, V), np.uint8)
    s = np.zeros(B, np.uint64)
    mean = np.zeros(B, np.float32)
    bad = lib().orc_uniform(ctypes.byref(d), *inst.tables(), int(fixed_gamma), float(inference_weight),
                            _p(alloc), _p(cfg), _p(s), _p(mean))
    if bad < 0:
        raise ValueError("oracle: invalid uniform arguments")
    return alloc, cfg, s, mean, int(bad)


def pareto(cost, post, with_bad=False):
    """Pareto-frontier mask (bit k = config k) of each set of configs (reading PR1); with
    with_bad, also the number of invalid sets (R-ERR, mask 0)."""
    cost = _c(cost, np.float32)
    post = _c(post, np.float32)
    n = cost.shape[-1]
    sets = cost.size // max(1, n)
    m = np.zeros(cost.shape[:-1], np.uint32)
    bad = lib().orc_pareto(sets, n, _p(cost), _p(post), _p(m))
    if bad < 0:
        raise ValueError("oracle: invalid pareto shape")
    return (m, int(bad)) if with_bad else m


def prune(cost, hist_acc, margin):
    """History-based pruning (readings PN1-PN3): cost [Q][n], hist_acc [Q][H][n] (NaN =
    unmeasured) -> keep mask [Q] (bit k = config k kept), number of invalid queries."""
    cost = _c(cost, np.float32)
    hist_acc = _c(hist_acc, np.float32)
    Q, n = cost.shape
    H = hist_acc.shape[1]
    assert hist_acc.shape == (Q, H, n)
    keep = np.zeros(Q, np.uint32)
    bad = lib().orc_prune(Q, H, n, _p(cost), _p(hist_acc), float(margin), _p(keep))
    if bad < 0:
        raise ValueError("oracle: invalid prune arguments")
    return keep, int(bad)


def curve_fit(acc, full_epochs):
    """Micro-profiler curve fit (readings CF1-CF3): acc [S][P] at epochs 1..P, full_epochs
    [S] -> predicted accuracy [S], params [S][3] = (alpha, c, beta2), bad."""
    acc = _c(acc, np.float32)
    S, Pn = acc.shape
    ke = _c(full_epochs, np.int32).reshape(S)
    pred = np.zeros(S, np.float32)
    prm = np.zeros((S, 3), np.float32)
    bad = lib().orc_curve_fit(S, Pn, _p(acc), _p(ke), _p(pred), _p(prm))
    if bad < 0:
        raise ValueError("oracle: invalid curve-fit shape")
    return pred, prm, int(bad)


def window(inst: Instances, mode: int = STEEPEST):
    """The retraining window as a timeline with the thief re-invoked at each completion
    (readings W1-W6): realized window-average accuracy [B], invocations [B], completion
    time per stream [B][V] (1 = none), bad."""
    d = inst.dims()
    B, V = inst.B, inst.V
    avg = np.zeros(B, np.float32)
    ev = np.zeros(B, np.uint32)
    done = np.zeros((B, V), np.float32)
    bad = lib().orc_window(ctypes.byref(d), *inst.tables(), int(mode), _p(avg), _p(ev), _p(done))
    if bad < 0:
        raise ValueError("oracle: invalid window arguments")
    return avg, ev, done, int(bad)
