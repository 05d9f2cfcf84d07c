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


class RecordLayout:
    """Chunked decision records for a gather that overlaps compute ("split the
    batch into >= 8 chunks and gather chunk i while computing chunk i+1").

    Every rank's instances [lo_r, hi_r) (shard_range of n_total) are split into n_chunks
    chunks of `chunk_inst` = ceil(B_max / n_chunks) instances; chunk c of a rank covers its
    local instances [c*chunk_inst, min(B_r, (c+1)*chunk_inst)).  A rank's buffer is its
    chunks back to back, each a record block of chunk_inst instances (record_views layout,
    unused rows zero-padded).  The gather of chunk c puts every rank's chunk-c block into the
    root's chunk-c region, rank-major: root_buf = [chunk 0: rank 0 .. rank P-1][chunk 1: ...]."""

    def __init__(self, n_total: int, nranks: int, n_streams: int, n_chunks: int = 1):
        self.n_total, self.nranks, self.V = n_total, nranks, n_streams
        self.per = [shard_range(n_total, nranks, r)[1] - shard_range(n_total, nranks, r)[0] for r in range(nranks)]
        bmax = max(self.per) if self.per else 0
        self.n_chunks = max(1, min(n_chunks, bmax)) if bmax else 1
        self.chunk_inst = -(-bmax // self.n_chunks) if bmax else 0
        self.chunk_bytes = record_bytes(self.chunk_inst, n_streams)
        self.rank_bytes = self.n_chunks * self.chunk_bytes
        self.root_bytes = self.nranks * self.rank_bytes

    def chunk_range(self, rank: int, c: int):
        """Local instance range [b0, b1) of chunk c on `rank` (may be empty)."""
        b0 = min(self.per[rank], c * self.chunk_inst)
        return b0, min(self.per[rank], b0 + self.chunk_inst)

    def local_chunk(self, buf: torch.Tensor, c: int) -> torch.Tensor:
        return buf[c * self.chunk_bytes:(c + 1) * self.chunk_bytes]

    def views(self, buf: torch.Tensor, rank: int, c: int):
        """Typed views of chunk c's valid rows in a rank buffer (kernels write straight into them)."""
        b0, b1 = self.chunk_range(rank, c)
        v = record_views(self.local_chunk(buf, c), self.chunk_inst, self.V)
        return {k: x[:b1 - b0] for k, x in v.items()}

    def root_chunk(self, root_buf: torch.Tensor, c: int) -> torch.Tensor:
        n = self.nranks * self.chunk_bytes
        return root_buf[c * n:(c + 1) * n]

    def unpack(self, root_buf: torch.Tensor):
        """Global instance order (rank 0's instances first, each rank's chunks in order)."""
        parts = {k: [] for k in ("sum", "mean", "steps", "alloc", "cfg")}
        for r in range(self.nranks):
            for c in range(self.n_chunks):
                b0, b1 = self.chunk_range(r, c)
                if b1 <= b0:
                    continue
                blk = self.root_chunk(root_buf, c)[r * self.chunk_bytes:(r + 1) * self.chunk_bytes]
                v = record_views(blk, self.chunk_inst, self.V)
                for k in parts:
                    parts[k].append(v[k][:b1 - b0])
        return {k: torch.cat(p) if p else torch.empty(0) for k, p in parts.items()}


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
