"""Instance sharding and decision records for the multi-GPU path.

Scheduling instances are independent (each is one window of one edge server,
P:1022), so rank r of P owns the contiguous block of instances
[r*ceil(B/P), min(B, (r+1)*ceil(B/P))) and computes it with no collective.  The
only exchange is the final gather of fixed-size decision records to the root
(ekya_gather_decisions / ncclGather).  A rank's record buffer is SoA:

    sum_q32 u64[B_r] | mean f32[B_r] | steps u32[B_r] | alloc u16[B_r][2V] | cfg u8[B_r][V]

i.e. 16 + 5V bytes per instance (66 B at V=10, 516 B at V=100), block padded to 16 B.  The root's
buffer is the P rank buffers back to back; ``unpack_root`` reassembles global
instance order.
"""
from __future__ import annotations

import torch


def shard_range(total: int, nranks: int, rank: int):
    per = -(-total // nranks)
    lo = min(total, rank * per)
    return lo, min(total, lo + per)


def record_bytes(n_inst: int, n_streams: int) -> int:
    """Bytes of one rank's record block, padded to 16 so blocks stay aligned at the root."""
    raw = n_inst * (8 + 4 + 4 + 4 * n_streams + n_streams)
    return (raw + 15) & ~15


def record_views(buf: torch.Tensor, n_inst: int, n_streams: int):
    """Typed views (sum, mean, steps, alloc, cfg) into a uint8 record buffer."""
    B, V, J = n_inst, n_streams, 2 * n_streams
    assert buf.dtype == torch.uint8 and buf.numel() >= record_bytes(B, V)
    o = 0
    out = {}
    for name, nbytes, dt, shape in (("sum", 8 * B, torch.uint64, (B,)), ("mean", 4 * B, torch.float32, (B,)),
                                    ("steps", 4 * B, torch.uint32, (B,)),
                                    ("alloc", 2 * J * B, torch.uint16, (B, J)),
                                    ("cfg", V * B, torch.uint8, (B, V))):
        out[name] = buf[o:o + nbytes].view(dt).view(shape)
        o += nbytes
    return out


def unpack_root(root_buf: torch.Tensor, nranks: int, n_inst_per_rank, n_streams: int):
    """Concatenate the per-rank records (in rank order) into global arrays.

    n_inst_per_rank: list of B_r (a rank's record block is record_bytes(B_max, V)
    long, padded when B_r < B_max so every rank sends the same byte count)."""
    bmax = max(n_inst_per_rank)
    rb = record_bytes(bmax, n_streams)
    parts = {k: [] for k in ("sum", "mean", "steps", "alloc", "cfg")}
    for r in range(nranks):
        v = record_views(root_buf[r * rb:(r + 1) * rb], bmax, n_streams)
        for k in parts:
            parts[k].append(v[k][:n_inst_per_rank[r]])
    return {k: torch.cat(p) for k, p in parts.items()}
