"""Seeded synthetic inputs for Ekya's scheduling hot path (shared by oracle and CUDA tests).

This module holds NONE of the method's arithmetic: it only draws instances.  It
is the one module both sides use ("input recipe").

Every value is a pure function of (seed, field, indices) through a counter-based
32-bit hash (lowbias32 finaliser), and every float is built with single IEEE
operations (+, -, *, /, floor, clamp; no libm transcendentals and no
order-dependent reductions), so the same call yields the same bits on the CPU
and on a CUDA device.  Multiplications modulo 2^32 are split into 16-bit halves
so no int64 product ever overflows.

Workload shapes follow the paper (SURVEY.md 8(d) / DESIGN.md 6):
  * scheduling instances: V streams, |Gamma| retraining configs with a 200x
    spread of GPU cost and post-retraining accuracy that usually but not
    always grows with cost, |Lambda| inference configs as frame-sampling
    levels whose accuracy factor shrinks with the sampling rate,
    stale accuracies 0.5-0.9, delta = Delta = 0.1 GPU,
    ||T|| = 200 s;
  * profiler queries: 27-class histograms (Waymo-shaped), 500 history windows
    ("10s to 100s"), 70 % of windows drawn around 5 cluster centres.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

MASK32 = 0xFFFFFFFF

# field ids (each random quantity draws from its own counter stream)
F_STALE, F_DEMAND, F_BETA, F_GMAX, F_COST, F_NOISE1, F_NOISE2, F_NOISE3 = range(1, 9)
F_LMU0, F_RHO, F_ALLOC, F_CENTRE, F_WTYPE, F_WCL, F_WN, F_BG, F_BASE, F_OFF = range(9, 19)
F_ANOISE1, F_ANOISE2, F_ANOISE3, F_SPARSE, F_WN2, F_PADG, F_PADL = range(19, 26)


def _mul32(x, m: int):
    """(x * m) mod 2^32 for x in [0, 2^32) without int64 overflow."""
    lo, hi = m & 0xFFFF, m >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & MASK32


def _mix(x):
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _hash(seed: int, fid: int, idx, device):
    h = _mix((seed * 0x9E3779B1 + fid * 0x85EBCA77) & MASK32)
    h = _mix(h ^ 0x5BD1E995)
    out = None
    for i in idx:
        if not torch.is_tensor(i):
            i = torch.tensor(int(i), dtype=torch.int64, device=device)
        i = i.to(torch.int64)
        assert True  # indices are < 2^32 by construction (checked by callers' shapes)
        base = h if out is None else out
        out = _mix(base ^ (i & MASK32))
    if out is None:
        out = torch.tensor(h, dtype=torch.int64, device=device)
    return out


def uniform(seed: int, fid: int, *idx, device="cpu"):
    """float32 in [0, 1) with 24 random bits, exact construction."""
    h = _hash(seed, fid, idx, device)
    return (h >> 8).to(torch.float32) * (1.0 / 16777216.0)


def _div(a, b):
    """IEEE a / b with b broadcast to a tensor: torch computes tensor / python-scalar
    as a reciprocal multiply on CUDA, which would break CPU/GPU bit-identity."""
    if not torch.is_tensor(b):
        b = torch.full_like(a, float(b))
    return a / b


def _ar(n, device):
    return torch.arange(n, dtype=torch.int64, device=device)


def _pow2_int(k):
    """Exact 2^k (float32) for integer-valued int64 tensor k in [-126, 127]."""
    return ((k + 127) << 23).to(torch.int32).view(torch.float32)


def _exp2_approx(e):
    """2^e for e >= 0 (float32): exact power of two times a cubic in the fraction."""
    k = torch.floor(e)
    fr = e - k
    poly = 1.0 + fr * (0.6951786 + fr * (0.2261370 + fr * 0.078125))
    return _pow2_int(k.to(torch.int64)) * poly


@dataclass
class SchedConfig:
    name: str
    n_streams: int
    n_gamma: int
    n_lambda: int
    units: int
    steal_units: int
    gpus: float
    delta_gpu: float
    window_s: float
    a_min: float
    n_inst: int
    seed: int
    kind: str = "cityscapes"          # "tiny" for config 1
    rho: tuple = (1.0, 0.75, 0.5, 0.25, 0.1)
    ragged: bool = False              # pad |Gamma_v|, |Lambda_v| per stream (sentinels)
    n_alloc: int = 0                  # LIST rows per instance

    @property
    def unit_gpu_seconds(self) -> float:
        return float(torch.tensor(self.delta_gpu * self.window_s, dtype=torch.float32))


# BASELINE.json configs
CONFIG1 = SchedConfig("tiny-2x2x2-U10", 2, 2, 2, 10, 1, 3.0, 0.3, 120.0, 0.40, 10000, 1001, kind="tiny")
CONFIG2 = SchedConfig("cityscapes-10x18x5-U80", 10, 18, 5, 80, 1, 8.0, 0.1, 200.0, 0.40, 4096, 2002)
CONFIG4 = SchedConfig("batch-65536x(10x18x5-U80)", 10, 18, 5, 80, 1, 8.0, 0.1, 200.0, 0.40, 65536, 4004,
                      n_alloc=4096)
CONFIG5 = SchedConfig("scaleout-100x18x5-U800", 100, 18, 5, 800, 1, 80.0, 0.1, 200.0, 0.40, 1000000, 5005)


def sched_tables(cfg: SchedConfig, lo: int = 0, hi: int | None = None, device="cpu"):
    """Tables for instances [lo, hi) of cfg, as torch tensors on `device`.

    Returns dict(stale [B,V] f32, cost/post [B,V,nG] f32, lam_min_units [B,V,nL] u16,
    lam_factor [B,V,nL] f32)."""
    hi = cfg.n_inst if hi is None else hi
    B, V, G, L = hi - lo, cfg.n_streams, cfg.n_gamma, cfg.n_lambda
    s = cfg.seed
    b = (_ar(B, device) + lo).view(B, 1, 1)
    v = _ar(V, device).view(1, V, 1)
    g = _ar(G, device).view(1, 1, G)
    lam = _ar(L, device).view(1, 1, L)
    uT = cfg.unit_gpu_seconds
    u = lambda f, *i: uniform(s, f, *i, device=device)

    stale = 0.5 + 0.4 * u(F_STALE, b, v)                       # [B,V,1]
    if cfg.kind == "tiny":
        cost = 40.0 + 50.0 * u(F_COST, b, v, g)
        post = torch.clamp(stale + (-0.05 + 0.4 * u(F_NOISE1, b, v, g)), 0.0, 1.0)
        rho = 0.5 + 0.4 * u(F_RHO, b, v)
        lf = torch.where(lam == 0, torch.ones_like(rho), rho).expand(B, V, L).clone()
        lmu0 = 2.0 + torch.floor(4.0 * u(F_LMU0, b, v))
        lmu = torch.where(lam == 0, lmu0, torch.ones_like(lmu0)).expand(B, V, L).clone()
    else:
        demand = 0.2 + 0.4 * u(F_DEMAND, b, v)                   # GPUs at full frame rate
        beta = 0.7 * u(F_BETA, b, v)
        gmax = 0.35 * u(F_GMAX, b, v)
        # cost: log-uniform over a 200x spread: uT * 0.25 * 200^u
        e = u(F_COST, b, v, g) * 7.643856
        cost = (uT * 0.25) * _exp2_approx(e)
        x = _div(cost, uT * 10.0)
        gain = gmax * _div(x, 1.0 + x)
        noise = (u(F_NOISE1, b, v, g) + u(F_NOISE2, b, v, g) + u(F_NOISE3, b, v, g) - 1.5) * 0.04
        post = torch.clamp((stale + gain) + noise, 0.0, 1.0)
        rho = torch.tensor(list(cfg.rho)[:L], dtype=torch.float32, device=device).view(1, 1, L)
        lf = rho + (1.0 - rho) * beta
        lmu = torch.floor(_div(rho * demand, cfg.delta_gpu)) + 1.0
    stale = stale.view(B, V)
    cost = cost.expand(B, V, G).contiguous()
    post = post.expand(B, V, G).contiguous()
    lf = lf.expand(B, V, L).contiguous()
    lmu = lmu.expand(B, V, L).contiguous()
    if cfg.ragged:
        # |Gamma_v| in [0, G], |Lambda_v| in [1, L]; padding sentinels
        ng = torch.floor(u(F_PADG, b, v) * (G + 1))
        nl = 1.0 + torch.floor(u(F_PADL, b, v) * L)
        cost = torch.where(g.to(torch.float32) >= ng, torch.full_like(cost, float("inf")), cost)
        lmu = torch.where(lam.to(torch.float32) >= nl, torch.full_like(lmu, 65535.0), lmu)
    return dict(stale=stale.contiguous(), cost=cost, post=post,
                lam_min_units=lmu.to(torch.int32).to(torch.uint16), lam_factor=lf)


def list_allocs(cfg: SchedConfig, n_alloc: int, lo: int = 0, hi: int | None = None, device="cpu"):
    """Random full allocations (sum == U) for LIST mode: [B, n_alloc, J] u16.

    Integer-only: weights w_j in [1, 2^16], parts floor(U w_j / sum w), leftover
    units to the lowest-numbered jobs."""
    hi = cfg.n_inst if hi is None else hi
    B, J, U = hi - lo, 2 * cfg.n_streams, cfg.units
    b = (_ar(B, device) + lo).view(B, 1, 1)
    n = _ar(n_alloc, device).view(1, n_alloc, 1)
    j = _ar(J, device).view(1, 1, J)
    w = (_hash(cfg.seed, F_ALLOC, (b, n, j), device) >> 16) + 1
    tot = torch.zeros_like(w[..., :1])
    for jj in range(J):
        tot = tot + w[..., jj:jj + 1]
    parts = (U * w) // tot
    used = torch.zeros_like(tot)
    for jj in range(J):
        used = used + parts[..., jj:jj + 1]
    parts = parts + (j < (U - used)).to(torch.int64)
    return parts.to(torch.int32).to(torch.uint16)


@dataclass
class ProfileConfig:
    name: str
    n_query: int
    n_hist: int
    n_class: int
    n_gamma: int
    tau: float = 0.2
    k: int = 5
    max_iter: int = 100
    seed: int = 3003
    frac_clustered: float = 0.7
    n_centres: int = 5
    sparse: bool = False


CONFIG3 = ProfileConfig("waymo-27c-500h-18g", 65536, 500, 27, 18)


def _rowsum(x):
    """Sequential (deterministic-order) sum over the last dim."""
    s = x[..., 0]
    for c in range(1, x.shape[-1]):
        s = s + x[..., c]
    return s


def profile_inputs(cfg: ProfileConfig, lo: int = 0, hi: int | None = None, device="cpu"):
    """cur [Q,C], hist [Q,H,C], hist_acc [Q,H,G] (NaN = unmeasured), fallback [Q,G]."""
    hi = cfg.n_query if hi is None else hi
    Q, H, C, G, K = hi - lo, cfg.n_hist, cfg.n_class, cfg.n_gamma, cfg.n_centres
    s = cfg.seed
    u = lambda f, *i: uniform(s, f, *i, device=device)
    q = (_ar(Q, device) + lo)
    # cluster centres per query: normalise(u^4), a sparse-ish simplex point
    qc = q.view(Q, 1, 1)
    ci = _ar(K, device).view(1, K, 1)
    cc = _ar(C, device).view(1, 1, C)
    r = u(F_CENTRE, qc, ci, cc)
    r = r * r
    r = r * r
    centres = _div(r, _rowsum(r).unsqueeze(-1).expand_as(r))                       # [Q,K,C]

    def windows(hidx):                                           # hidx [1,W] -> [Q,W,C], cluster id
        W = hidx.shape[1]
        qh = q.view(Q, 1)
        clustered = u(F_WTYPE, qh, hidx) < cfg.frac_clustered      # [Q,W]
        cl = torch.floor(u(F_WCL, qh, hidx) * K).to(torch.int64).clamp_(0, K - 1)
        cen = torch.gather(centres, 1, cl.unsqueeze(-1).expand(Q, W, C))
        q3, h3, c3 = q.view(Q, 1, 1), hidx.view(1, W, 1), cc
        raw_c = cen * (0.75 + 0.5 * u(F_WN, q3, h3, c3)) + 0.002 * u(F_WN2, q3, h3, c3)
        bg = u(F_BG, q3, h3, c3)
        raw_b = bg * bg * bg
        raw = torch.where(clustered.unsqueeze(-1), raw_c, raw_b)
        hist = _div(raw, _rowsum(raw).unsqueeze(-1).expand_as(raw))
        label = torch.where(clustered, cl, K + hidx.expand(Q, W))
        return hist, label

    hist, label = windows(_ar(H, device).view(1, H))
    cur, _ = windows(torch.full((1, 1), H, dtype=torch.int64, device=device))
    cur = cur.view(Q, C)
    gq = _ar(G, device)
    base = 0.5 + 0.4 * u(F_BASE, q.view(Q, 1), gq.view(1, G))   # [Q,G]
    l3 = label.view(Q, H, 1)
    off = 0.2 * (u(F_OFF, q.view(Q, 1, 1), l3, gq.view(1, 1, G)) - 0.5)
    q3, h3, g3 = q.view(Q, 1, 1), _ar(H, device).view(1, H, 1), gq.view(1, 1, G)
    nz = (u(F_ANOISE1, q3, h3, g3) + u(F_ANOISE2, q3, h3, g3) + u(F_ANOISE3, q3, h3, g3) - 1.5) * 0.04
    acc = torch.clamp((base.view(Q, 1, G) + off) + nz, 0.0, 1.0)
    if cfg.sparse:
        pick = torch.floor(u(F_SPARSE, q.view(Q, 1), _ar(H, device).view(1, H)) * G).to(torch.int64)
        acc = torch.where(g3 == pick.view(Q, H, 1), acc, torch.full_like(acc, float("nan")))
    return dict(cur=cur.contiguous(), hist=hist.contiguous(), hist_acc=acc.contiguous(),
                fallback=base.contiguous())
