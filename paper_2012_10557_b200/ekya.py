"""Thin Python binding of libekya (include/ekya.h): argument marshalling only.

Every function forwards torch tensors' device pointers and the current CUDA
stream to the C ABI of the same name; every step of the hot path runs in the
sm_100a kernels of ``libekya.so``.  There is no CPU fallback: if the library is
missing or a tensor is not a contiguous CUDA tensor of the documented dtype,
this module raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libekya.so")

EKYA_OK = 0
ERRORS = {-1: "EKYA_ERR_ARG", -2: "EKYA_ERR_LIMIT", -3: "EKYA_ERR_SHAPE", -4: "EKYA_ERR_CUDA",
          -5: "EKYA_ERR_NCCL", -6: "EKYA_ERR_DATA"}
EVAL_LIST, EVAL_GRID = 0, 1
THIEF_STEEPEST, THIEF_LITERAL = 0, 1
PROFILE_RADIUS, PROFILE_CLUSTER = 0, 1
LAMBDA_NONE = 7
SYMBOLS = ["ekya_create", "ekya_destroy", "ekya_last_error", "ekya_launch_count", "ekya_version",
           "ekya_eval_allocations", "ekya_thief_schedule", "ekya_profile_estimate", "ekya_profile_estimate_both",
           "ekya_comm_unique_id", "ekya_comm_init", "ekya_comm_info", "ekya_gather_decisions", "ekya_counters", "ekya_place",
           "ekya_checkpoint_decide", "ekya_uniform_schedule", "ekya_pareto", "ekya_prune_configs", "ekya_curve_fit",
           "ekya_window_workspace_bytes", "ekya_window_schedule"]


class EkyaError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"{what} failed: {ERRORS.get(code, code)}")
        self.code = code


class Dims(ctypes.Structure):
    """ekya_dims (include/ekya.h)."""
    _fields_ = [("n_inst", ctypes.c_int32), ("n_streams", ctypes.c_int32),
                ("n_gamma", ctypes.c_int32), ("n_lambda", ctypes.c_int32),
                ("units", ctypes.c_int32), ("steal_units", ctypes.c_int32),
                ("unit_gpu_seconds", ctypes.c_float), ("a_min", ctypes.c_float)]


class Tables(ctypes.Structure):
    """ekya_tables: device pointers."""
    _fields_ = [("stale", ctypes.c_void_p), ("cost", ctypes.c_void_p), ("post", ctypes.c_void_p),
                ("lam_min_units", ctypes.c_void_p), ("lam_factor", ctypes.c_void_p)]


class ProfileDims(ctypes.Structure):
    _fields_ = [("n_query", ctypes.c_int32), ("n_hist", ctypes.c_int32),
                ("n_class", ctypes.c_int32), ("n_gamma", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("tau", ctypes.c_float),
                ("k", ctypes.c_int32), ("max_iter", ctypes.c_int32)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libekya.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libekya.so not built at {path}; run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    P, I32, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64
    L.ekya_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, ctypes.c_size_t]
    L.ekya_create.restype = ctypes.c_int
    L.ekya_destroy.argtypes = [P]
    L.ekya_destroy.restype = None
    L.ekya_last_error.argtypes = [P]
    L.ekya_last_error.restype = ctypes.c_int
    L.ekya_launch_count.argtypes = [P]
    L.ekya_launch_count.restype = U64
    L.ekya_counters.argtypes = [P, P, ctypes.c_int]
    L.ekya_counters.restype = ctypes.c_int
    L.ekya_version.argtypes = []
    L.ekya_version.restype = ctypes.c_char_p
    L.ekya_eval_allocations.argtypes = [P, ctypes.POINTER(Dims), ctypes.POINTER(Tables), ctypes.c_int,
                                        I32, P, P, P, P, P, P, P]
    L.ekya_eval_allocations.restype = ctypes.c_int
    L.ekya_thief_schedule.argtypes = [P, ctypes.POINTER(Dims), ctypes.POINTER(Tables), ctypes.c_int,
                                      P, P, P, P, P, P]
    L.ekya_thief_schedule.restype = ctypes.c_int
    L.ekya_profile_estimate.argtypes = [P, ctypes.POINTER(ProfileDims), P, P, P, P, P, P, P, P]
    L.ekya_profile_estimate.restype = ctypes.c_int
    L.ekya_profile_estimate_both.argtypes = [P, ctypes.POINTER(ProfileDims), P, P, P, P, P, P, P, P, P, P]
    L.ekya_profile_estimate_both.restype = ctypes.c_int
    L.ekya_uniform_schedule.argtypes = [P, ctypes.POINTER(Dims), ctypes.POINTER(Tables), ctypes.c_int32,
                                        ctypes.c_float, P, P, P, P, P]
    L.ekya_uniform_schedule.restype = ctypes.c_int
    L.ekya_pareto.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, P, P, P]
    L.ekya_pareto.restype = ctypes.c_int
    L.ekya_prune_configs.argtypes = [P, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, P, P, ctypes.c_float, P, P]
    L.ekya_prune_configs.restype = ctypes.c_int
    L.ekya_window_workspace_bytes.argtypes = [ctypes.POINTER(Dims)]
    L.ekya_window_workspace_bytes.restype = ctypes.c_size_t
    L.ekya_window_schedule.argtypes = [P, ctypes.POINTER(Dims), ctypes.POINTER(Tables), ctypes.c_int, P,
                                       ctypes.c_size_t, P, P, P, P]
    L.ekya_window_schedule.restype = ctypes.c_int
    L.ekya_curve_fit.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, P, P, P, P]
    L.ekya_curve_fit.restype = ctypes.c_int
    L.ekya_place.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P, P, P, P, P, P]
    L.ekya_place.restype = ctypes.c_int
    L.ekya_checkpoint_decide.argtypes = [P, ctypes.c_int64] + [P] * 8 + [P]
    L.ekya_checkpoint_decide.restype = ctypes.c_int
    L.ekya_comm_unique_id.argtypes = [P]
    L.ekya_comm_unique_id.restype = ctypes.c_int
    L.ekya_comm_init.argtypes = [P, P, ctypes.c_int, ctypes.c_int]
    L.ekya_comm_init.restype = ctypes.c_int
    L.ekya_comm_info.argtypes = [P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    L.ekya_comm_info.restype = ctypes.c_int
    L.ekya_gather_decisions.argtypes = [P, P, ctypes.c_size_t, P, ctypes.c_int, P]
    L.ekya_gather_decisions.restype = ctypes.c_int
    _lib = L
    return L


def _check(code, what):
    if code != EKYA_OK:
        raise EkyaError(code, what)


def _ptr(t, dtype, name, optional=False, numel=None):
    """Device pointer of a contiguous CUDA tensor of `dtype`; with `numel`, the tensor must
    hold exactly that many elements (the count the C call will read or write)."""
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name} is required")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must hold {numel} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr()) if t.numel() else None


def _stream(stream, h=None):
    """The stream to launch on: the given one, else the current stream of the handle's device.
    A stream on another device than the handle's is rejected."""
    dev = h.device if h is not None else None
    s = (torch.cuda.current_stream(dev) if dev is not None else torch.cuda.current_stream()) \
        if stream is None else stream
    if dev is not None and s.device.index is not None and s.device.index != dev:
        raise ValueError(f"stream is on cuda:{s.device.index}, the handle on cuda:{dev}")
    return ctypes.c_void_p(s.cuda_stream)


class Handle:
    """Owns an ekya_handle (device error word + launch counter + optional NCCL comm)."""

    def __init__(self, device: int | None = None):
        L = load_library()
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = dev
        h = ctypes.c_void_p()
        _check(L.ekya_create(ctypes.byref(h), dev, 0), "ekya_create")
        self._h = h

    @property
    def ptr(self):
        return self._h

    def close(self):
        if self._h:
            load_library().ekya_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> int:
        return load_library().ekya_last_error(self._h)

    def launch_count(self) -> int:
        return int(load_library().ekya_launch_count(self._h))

    def counters(self) -> dict:
        buf = (ctypes.c_uint64 * 2)()
        _check(load_library().ekya_counters(self._h, ctypes.cast(buf, ctypes.c_void_p), 2), "ekya_counters")
        return {"launches": int(buf[0]), "lloyd_passes": int(buf[1])}


def make_dims(n_inst, n_streams, n_gamma, n_lambda, units, steal_units, unit_gpu_seconds, a_min):
    return Dims(n_inst, n_streams, n_gamma, n_lambda, units, steal_units, unit_gpu_seconds, a_min)


def make_tables(stale, cost, post, lam_min_units, lam_factor):
    """Device tables; keep the tensors alive while the returned struct is in use.  The
    element counts are remembered and checked against the dims of every call."""
    t = Tables(_ptr(stale, torch.float32, "stale"), _ptr(cost, torch.float32, "cost", True),
               _ptr(post, torch.float32, "post", True),
               _ptr(lam_min_units, torch.uint16, "lam_min_units"),
               _ptr(lam_factor, torch.float32, "lam_factor"))
    t.numels = (stale.numel(), cost.numel(), post.numel(), lam_min_units.numel(), lam_factor.numel())
    return t


def _check_tables(dims, tables):
    BV = dims.n_inst * dims.n_streams
    want = (BV, BV * dims.n_gamma, BV * dims.n_gamma, BV * dims.n_lambda, BV * dims.n_lambda)
    got = getattr(tables, "numels", None)
    if got is not None and tuple(got) != want:
        raise ValueError(f"tables hold {got} elements, dims need {want} (stale, cost, post, lam_min_units, "
                         "lam_factor)")


def dims_from(tables: dict, units, steal_units, unit_gpu_seconds, a_min):
    B, V = tables["stale"].shape
    return make_dims(B, V, tables["cost"].shape[2], tables["lam_factor"].shape[2], units, steal_units,
                     unit_gpu_seconds, a_min)


# ---------------------------------------------------------------------------
# C-ABI entry points (same names)
# ---------------------------------------------------------------------------
def ekya_eval_allocations(h: Handle, dims: Dims, tables: Tables, mode: int, n_alloc=0, alloc=None,
                          out_sum_q32=None, out_mean=None, out_cfg=None, out_grid=None,
                          out_grid_cfg=None, stream=None):
    L = load_library()
    _check_tables(dims, tables)
    B, V = dims.n_inst, dims.n_streams
    nl = B * n_alloc if mode == EVAL_LIST else None
    ng = B * V * n_cells(dims.units) if mode == EVAL_GRID else None
    code = L.ekya_eval_allocations(
        h.ptr, ctypes.byref(dims), ctypes.byref(tables), mode, n_alloc,
        _ptr(alloc, torch.uint16, "alloc", True, nl and nl * 2 * V),
        _ptr(out_sum_q32, torch.uint64, "out_sum_q32", True, nl),
        _ptr(out_mean, torch.float32, "out_mean", True, nl), _ptr(out_cfg, torch.uint8, "out_cfg", True, nl and nl * V),
        _ptr(out_grid, torch.float32, "out_grid", True, ng),
        _ptr(out_grid_cfg, torch.uint8, "out_grid_cfg", True, ng), _stream(stream, h))
    _check(code, "ekya_eval_allocations")


def ekya_thief_schedule(h: Handle, dims: Dims, tables: Tables, mode: int, out_alloc, out_cfg,
                        out_sum_q32, out_mean=None, out_steps=None, stream=None):
    L = load_library()
    _check_tables(dims, tables)
    B, V = dims.n_inst, dims.n_streams
    code = L.ekya_thief_schedule(h.ptr, ctypes.byref(dims), ctypes.byref(tables), mode,
                                 _ptr(out_alloc, torch.uint16, "out_alloc", numel=2 * B * V),
                                 _ptr(out_cfg, torch.uint8, "out_cfg", numel=B * V),
                                 _ptr(out_sum_q32, torch.uint64, "out_sum_q32", numel=B),
                                 _ptr(out_mean, torch.float32, "out_mean", True, B),
                                 _ptr(out_steps, torch.uint32, "out_steps", True, B), _stream(stream, h))
    _check(code, "ekya_thief_schedule")


def ekya_profile_estimate(h: Handle, pdims: ProfileDims, cur, hist, hist_acc, fallback, out_est,
                          out_n, out_cluster=None, stream=None):
    L = load_library()
    Q, H, C, G = pdims.n_query, pdims.n_hist, pdims.n_class, pdims.n_gamma
    code = L.ekya_profile_estimate(h.ptr, ctypes.byref(pdims), _ptr(cur, torch.float32, "cur", numel=Q * C),
                                   _ptr(hist, torch.float32, "hist", True, Q * H * C),
                                   _ptr(hist_acc, torch.float32, "hist_acc", True, Q * H * G),
                                   _ptr(fallback, torch.float32, "fallback", numel=Q * G),
                                   _ptr(out_est, torch.float32, "out_est", numel=Q * G),
                                   _ptr(out_n, torch.int32, "out_n", numel=Q * G),
                                   _ptr(out_cluster, torch.int32, "out_cluster", True, Q * (H + 1)),
                                   _stream(stream, h))
    _check(code, "ekya_profile_estimate")


def ekya_profile_estimate_both(h: Handle, pdims: ProfileDims, cur, hist, hist_acc, fallback, out_est_radius,
                               out_n_radius, out_est_cluster, out_n_cluster, out_cluster=None, stream=None):
    L = load_library()
    Q, H, C, G = pdims.n_query, pdims.n_hist, pdims.n_class, pdims.n_gamma
    code = L.ekya_profile_estimate_both(h.ptr, ctypes.byref(pdims), _ptr(cur, torch.float32, "cur", numel=Q * C),
                                        _ptr(hist, torch.float32, "hist", True, Q * H * C),
                                        _ptr(hist_acc, torch.float32, "hist_acc", True, Q * H * G),
                                        _ptr(fallback, torch.float32, "fallback", numel=Q * G),
                                        _ptr(out_est_radius, torch.float32, "out_est_radius", numel=Q * G),
                                        _ptr(out_n_radius, torch.int32, "out_n_radius", numel=Q * G),
                                        _ptr(out_est_cluster, torch.float32, "out_est_cluster", numel=Q * G),
                                        _ptr(out_n_cluster, torch.int32, "out_n_cluster", numel=Q * G),
                                        _ptr(out_cluster, torch.int32, "out_cluster", True, Q * (H + 1)),
                                        _stream(stream, h))
    _check(code, "ekya_profile_estimate_both")


def ekya_uniform_schedule(h: Handle, dims: Dims, tables: Tables, fixed_gamma: int, inference_weight: float,
                          out_alloc, out_cfg, out_sum_q32, out_mean=None, stream=None):
    L = load_library()
    _check_tables(dims, tables)
    B, V = dims.n_inst, dims.n_streams
    code = L.ekya_uniform_schedule(h.ptr, ctypes.byref(dims), ctypes.byref(tables), int(fixed_gamma),
                                   float(inference_weight), _ptr(out_alloc, torch.uint16, "out_alloc", numel=2 * B * V),
                                   _ptr(out_cfg, torch.uint8, "out_cfg", numel=B * V),
                                   _ptr(out_sum_q32, torch.uint64, "out_sum_q32", numel=B),
                                   _ptr(out_mean, torch.float32, "out_mean", True, B), _stream(stream, h))
    _check(code, "ekya_uniform_schedule")


def ekya_pareto(h: Handle, cost, post, out_mask, stream=None):
    L = load_library()
    n = cost.shape[-1]
    n_sets = 1
    for x in cost.shape[:-1]:
        n_sets *= int(x)
    if tuple(post.shape) != tuple(cost.shape):
        raise ValueError("ekya_pareto: post must have cost's shape")
    code = L.ekya_pareto(h.ptr, n_sets, n, _ptr(cost, torch.float32, "cost", True),
                         _ptr(post, torch.float32, "post", True),
                         _ptr(out_mask, torch.uint32, "out_mask", numel=n_sets), _stream(stream, h))
    _check(code, "ekya_pareto")


def ekya_prune_configs(h: Handle, cost, hist_acc, margin: float, out_keep, stream=None):
    L = load_library()
    Q, n = cost.shape
    H = hist_acc.shape[1]
    if tuple(hist_acc.shape) != (Q, H, n) or tuple(out_keep.shape) != (Q,):
        raise ValueError("ekya_prune_configs: cost [Q][n], hist_acc [Q][H][n], out_keep [Q]")
    code = L.ekya_prune_configs(h.ptr, Q, H, n, _ptr(cost, torch.float32, "cost", True),
                                _ptr(hist_acc, torch.float32, "hist_acc", True), float(margin),
                                _ptr(out_keep, torch.uint32, "out_keep"), _stream(stream, h))
    _check(code, "ekya_prune_configs")


def ekya_window_workspace_bytes(dims: Dims) -> int:
    return int(load_library().ekya_window_workspace_bytes(ctypes.byref(dims)))


def ekya_window_schedule(h: Handle, dims: Dims, tables: Tables, mode: int, workspace, out_avg, out_events, out_done,
                         stream=None):
    L = load_library()
    _check_tables(dims, tables)
    B, V = dims.n_inst, dims.n_streams
    code = L.ekya_window_schedule(h.ptr, ctypes.byref(dims), ctypes.byref(tables), mode,
                                  _ptr(workspace, torch.uint8, "workspace"), workspace.numel(),
                                  _ptr(out_avg, torch.float32, "out_avg", numel=B),
                                  _ptr(out_events, torch.uint32, "out_events", numel=B),
                                  _ptr(out_done, torch.float32, "out_done", numel=B * V), _stream(stream, h))
    _check(code, "ekya_window_schedule")


def ekya_curve_fit(h: Handle, acc, full_epochs, out_pred, out_params=None, stream=None):
    L = load_library()
    S, n = acc.shape
    code = L.ekya_curve_fit(h.ptr, S, n, _ptr(acc, torch.float32, "acc"),
                            _ptr(full_epochs, torch.int32, "full_epochs", numel=S),
                            _ptr(out_pred, torch.float32, "out_pred", numel=S),
                            _ptr(out_params, torch.float32, "out_params", True, 3 * S), _stream(stream, h))
    _check(code, "ekya_curve_fit")


def ekya_place(h: Handle, units: int, gpus: int, alloc, out_piece_job, out_piece_q, out_piece_gpu, out_n_pieces,
               out_gpu_load=None, stream=None):
    L = load_library()
    B, J = alloc.shape
    P = B * (J + gpus)
    code = L.ekya_place(h.ptr, B, J, units, gpus, _ptr(alloc, torch.uint16, "alloc"),
                        _ptr(out_piece_job, torch.uint16, "out_piece_job", numel=P),
                        _ptr(out_piece_q, torch.uint32, "out_piece_q", numel=P),
                        _ptr(out_piece_gpu, torch.int16, "out_piece_gpu", numel=P),
                        _ptr(out_n_pieces, torch.uint16, "out_n_pieces", numel=B),
                        _ptr(out_gpu_load, torch.uint32, "out_gpu_load", True, B * gpus), _stream(stream, h))
    _check(code, "ekya_place")


def ekya_checkpoint_decide(h: Handle, tau, t, T, a, a_star, A, delta_ckpt, out, stream=None):
    L = load_library()
    n = out.numel()
    args = [_ptr(x, torch.float32, nm, numel=n) for x, nm in ((tau, "tau"), (t, "t"), (T, "T"), (a, "a"),
                                                              (a_star, "a_star"), (A, "A"), (delta_ckpt, "delta_ckpt"))]
    code = L.ekya_checkpoint_decide(h.ptr, n, *args, _ptr(out, torch.uint8, "out"), _stream(stream, h))
    _check(code, "ekya_checkpoint_decide")


def ekya_comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().ekya_comm_unique_id(buf), "ekya_comm_unique_id")
    return buf.raw


def ekya_comm_init(h: Handle, uid: bytes, nranks: int, rank: int):
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    _check(load_library().ekya_comm_init(h.ptr, buf, nranks, rank), "ekya_comm_init")


def ekya_comm_info(h: Handle):
    """(nranks, rank) of the handle's NCCL communicator (1, 0 without one)."""
    n, r = ctypes.c_int(), ctypes.c_int()
    _check(load_library().ekya_comm_info(h.ptr, ctypes.byref(n), ctypes.byref(r)), "ekya_comm_info")
    return n.value, r.value


def ekya_gather_decisions(h: Handle, local, root_buf, root=0, stream=None):
    if not local.is_cuda or not local.is_contiguous():
        raise ValueError("local must be a contiguous CUDA tensor")
    rb = None
    if root_buf is not None:
        if not root_buf.is_cuda or not root_buf.is_contiguous():
            raise ValueError("root_buf must be a contiguous CUDA tensor")
        rb = ctypes.c_void_p(root_buf.data_ptr())
    nbytes = local.numel() * local.element_size()
    _check(load_library().ekya_gather_decisions(h.ptr, ctypes.c_void_p(local.data_ptr()), nbytes, rb,
                                                root, _stream(stream, h)), "ekya_gather_decisions")


# ---------------------------------------------------------------------------
# convenience wrappers that allocate outputs (still marshalling only)
# ---------------------------------------------------------------------------
def n_cells(units: int) -> int:
    return (units + 1) * (units + 2) // 2


def eval_grid(h, tables: dict, units, steal_units, unit_gpu_seconds, a_min, with_cfg=True, stream=None):
    dims = dims_from(tables, units, steal_units, unit_gpu_seconds, a_min)
    B, V = dims.n_inst, dims.n_streams
    dev = tables["stale"].device
    grid = torch.empty((B, V, n_cells(units)), dtype=torch.float32, device=dev)
    gcfg = torch.empty((B, V, n_cells(units)), dtype=torch.uint8, device=dev) if with_cfg else None
    ekya_eval_allocations(h, dims, make_tables(**tables), EVAL_GRID, out_grid=grid, out_grid_cfg=gcfg,
                          stream=stream)
    return grid, gcfg


def eval_list(h, tables: dict, alloc, units, steal_units, unit_gpu_seconds, a_min, stream=None):
    dims = dims_from(tables, units, steal_units, unit_gpu_seconds, a_min)
    B, N, V = alloc.shape[0], alloc.shape[1], dims.n_streams
    dev = alloc.device
    s = torch.empty((B, N), dtype=torch.uint64, device=dev)
    mean = torch.empty((B, N), dtype=torch.float32, device=dev)
    cfg = torch.empty((B, N, V), dtype=torch.uint8, device=dev)
    ekya_eval_allocations(h, dims, make_tables(**tables), EVAL_LIST, N, alloc, s, mean, cfg,
                          stream=stream)
    return s, mean, cfg


def thief_schedule(h, tables: dict, units, steal_units, unit_gpu_seconds, a_min, mode=THIEF_STEEPEST,
                   stream=None):
    dims = dims_from(tables, units, steal_units, unit_gpu_seconds, a_min)
    B, V = dims.n_inst, dims.n_streams
    dev = tables["stale"].device
    alloc = torch.empty((B, 2 * V), dtype=torch.uint16, device=dev)
    cfg = torch.empty((B, V), dtype=torch.uint8, device=dev)
    s = torch.empty(B, dtype=torch.uint64, device=dev)
    mean = torch.empty(B, dtype=torch.float32, device=dev)
    steps = torch.empty(B, dtype=torch.uint32, device=dev)
    ekya_thief_schedule(h, dims, make_tables(**tables), mode, alloc, cfg, s, mean, steps, stream=stream)
    return alloc, cfg, s, mean, steps


def profile_estimate(h, cur, hist, hist_acc, fallback, mode=PROFILE_RADIUS, tau=0.2, k=5, max_iter=100,
                     with_cluster=False, stream=None):
    Q, C = cur.shape
    H = hist.shape[1]
    G = fallback.shape[1]
    pd = ProfileDims(Q, H, C, G, mode, tau, k, max_iter)
    est = torch.empty((Q, G), dtype=torch.float32, device=cur.device)
    n = torch.empty((Q, G), dtype=torch.int32, device=cur.device)
    cl = torch.empty((Q, H + 1), dtype=torch.int32, device=cur.device) if with_cluster else None
    ekya_profile_estimate(h, pd, cur, hist, hist_acc, fallback, est, n, cl, stream=stream)
    return est, n, cl


def profile_estimate_both(h, cur, hist, hist_acc, fallback, tau=0.2, k=5, max_iter=100, with_cluster=False,
                          stream=None):
    """RADIUS and CLUSTER estimates of the same queries in one call (one history pass for the
    paper's Waymo shape): (est_radius, n_radius, est_cluster, n_cluster, cluster)."""
    Q, C = cur.shape
    H = hist.shape[1]
    G = fallback.shape[1]
    pd = ProfileDims(Q, H, C, G, PROFILE_CLUSTER, tau, k, max_iter)
    er = torch.empty((Q, G), dtype=torch.float32, device=cur.device)
    nr = torch.empty((Q, G), dtype=torch.int32, device=cur.device)
    ec = torch.empty((Q, G), dtype=torch.float32, device=cur.device)
    nc = torch.empty((Q, G), dtype=torch.int32, device=cur.device)
    cl = torch.empty((Q, H + 1), dtype=torch.int32, device=cur.device) if with_cluster else None
    ekya_profile_estimate_both(h, pd, cur, hist, hist_acc, fallback, er, nr, ec, nc, cl, stream=stream)
    return er, nr, ec, nc, cl


def place(h, alloc, units, gpus, stream=None):
    """Placement of allocations (units) onto `gpus` GPUs; returns (piece_job, piece_q,
    piece_gpu, n_pieces, gpu_load) as device tensors (include/ekya.h ekya_place)."""
    B, J = alloc.shape
    dev = alloc.device
    P = J + gpus
    pj = torch.empty((B, P), dtype=torch.uint16, device=dev)
    pq = torch.empty((B, P), dtype=torch.uint32, device=dev)
    pg = torch.empty((B, P), dtype=torch.int16, device=dev)
    npc = torch.empty((B,), dtype=torch.uint16, device=dev)
    load = torch.empty((B, gpus), dtype=torch.uint32, device=dev)
    ekya_place(h, units, gpus, alloc, pj, pq, pg, npc, load, stream=stream)
    return pj, pq, pg, npc, load


def checkpoint_decide(h, tau, t, T, a, a_star, A, delta_ckpt, stream=None):
    out = torch.empty(tau.shape, dtype=torch.uint8, device=tau.device)
    ekya_checkpoint_decide(h, tau, t, T, a, a_star, A, delta_ckpt, out, stream=stream)
    return out


HIGHEST_POST = -1


def uniform_schedule(h, tables: dict, units, steal_units, unit_gpu_seconds, a_min, fixed_gamma=HIGHEST_POST,
                     inference_weight=0.5, stream=None):
    dims = dims_from(tables, units, steal_units, unit_gpu_seconds, a_min)
    B, V = dims.n_inst, dims.n_streams
    dev = tables["stale"].device
    alloc = torch.empty((B, 2 * V), dtype=torch.uint16, device=dev)
    cfg = torch.empty((B, V), dtype=torch.uint8, device=dev)
    s = torch.empty((B,), dtype=torch.uint64, device=dev)
    mean = torch.empty((B,), dtype=torch.float32, device=dev)
    ekya_uniform_schedule(h, dims, make_tables(**tables), fixed_gamma, inference_weight, alloc, cfg, s, mean,
                          stream=stream)
    return alloc, cfg, s, mean


def pareto(h, cost, post, stream=None):
    out = torch.empty(cost.shape[:-1], dtype=torch.uint32, device=cost.device)
    ekya_pareto(h, cost, post, out, stream=stream)
    return out


def prune_configs(h, cost, hist_acc, margin, stream=None):
    """History-based pruning (PN1-PN3): cost [Q][n], hist_acc [Q][H][n] -> keep mask [Q] u32."""
    out = torch.empty(cost.shape[:1], dtype=torch.uint32, device=cost.device)
    ekya_prune_configs(h, cost, hist_acc, margin, out, stream=stream)
    return out


def curve_fit(h, acc, full_epochs, stream=None):
    """Micro-profiler curve fit: acc [S][P] (epochs 1..P), full_epochs [S] int32 ->
    (predicted accuracy [S], params [S][3] = (alpha, c, beta2))."""
    S = acc.shape[0]
    pred = torch.empty((S,), dtype=torch.float32, device=acc.device)
    prm = torch.empty((S, 3), dtype=torch.float32, device=acc.device)
    ekya_curve_fit(h, acc, full_epochs, pred, prm, stream=stream)
    return pred, prm


def window_schedule(h, tables: dict, units, steal_units, unit_gpu_seconds, a_min, mode=THIEF_STEEPEST, stream=None):
    """The window timeline with re-invocation at completions: (avg [B], events [B], done [B][V])."""
    dims = dims_from(tables, units, steal_units, unit_gpu_seconds, a_min)
    B, V = dims.n_inst, dims.n_streams
    dev = tables["stale"].device
    ws = torch.empty((max(1, ekya_window_workspace_bytes(dims)),), dtype=torch.uint8, device=dev)
    avg = torch.empty((B,), dtype=torch.float32, device=dev)
    ev = torch.empty((B,), dtype=torch.uint32, device=dev)
    done = torch.empty((B, V), dtype=torch.float32, device=dev)
    ekya_window_schedule(h, dims, make_tables(**tables), mode, ws, avg, ev, done, stream=stream)
    return avg, ev, done
