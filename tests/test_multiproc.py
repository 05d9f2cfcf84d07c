"""World-size-2 gloo tests of the multi-GPU host logic (-m "not gpu").

Each rank generates ONLY its shard of the instances (synth keyed by global
instance id), computes decisions for it (here with the CPU oracle, standing in
for the device kernels the GPU path runs), packs them into the decision-record
layout of paper_2012_10557_b200.shard and gathers them to rank 0 -- the same
data movement ekya_gather_decisions performs with ncclGather.  Rank 0 must
reassemble records byte-identical to a single-process run over all instances.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2012_10557_b200 import shard


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decisions(cfg, lo, hi, mode):
    T = synth.sched_tables(cfg, lo, hi)
    inst = oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                            cfg.units, cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)
    return oracle.thief(inst, mode)


def _body(rank, world, total, mode, q, n_chunks):
    """The data plane of bench.py's chunked gather (shard.RecordLayout): each rank writes its
    chunk-c decisions into the chunk's typed record views, then chunk c is gathered to the
    root's chunk-c region (here dist.gather over gloo; on GPUs ekya_gather_decisions ->
    ncclGather with the same offsets), and the root unpacks global instance order."""
    cfg = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": total})
    lo, hi = shard.shard_range(total, world, rank)
    V = cfg.n_streams
    L = shard.RecordLayout(total, world, V, n_chunks)
    buf = torch.zeros(L.rank_bytes, dtype=torch.uint8)
    root = torch.zeros(L.root_bytes, dtype=torch.uint8) if rank == 0 else None
    for c in range(L.n_chunks):
        b0, b1 = L.chunk_range(rank, c)
        views = L.views(buf, rank, c)
        if b1 > b0:
            a, cf, s, m, st, _ = _decisions(cfg, lo + b0, lo + b1, mode)
            views["sum"][:] = torch.from_numpy(s.astype(np.uint64))
            views["mean"][:] = torch.from_numpy(m)
            views["steps"][:] = torch.from_numpy(st)
            views["alloc"][:] = torch.from_numpy(a)
            views["cfg"][:] = torch.from_numpy(cf)
        local = L.local_chunk(buf, c)
        gl = [torch.zeros_like(local) for _ in range(world)] if rank == 0 else None
        dist.gather(local, gl, dst=0)
        if rank == 0:
            L.root_chunk(root, c).copy_(torch.cat(gl))
    if rank == 0:
        got = L.unpack(root)
        q.put({k: v.numpy().copy() for k, v in got.items()})


def _worker(rank, world, port, total, mode, q, n_chunks=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, total, mode, q, n_chunks)
    except Exception as e:  # surface the failure instead of hanging the test
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total,mode,n_chunks", [(12, 0, 1), (11, 1, 1), (23, 0, 4), (9, 1, 8)])
def test_sharded_gather_equals_single_run(total, mode, n_chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, mode, q, n_chunks)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    assert isinstance(got, dict), got
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": total})
    a, c, s, m, st, _ = _decisions(cfg, 0, total, mode)
    assert np.array_equal(got["alloc"], a)
    assert np.array_equal(got["cfg"], c)
    assert np.array_equal(got["sum"], s)
    assert np.array_equal(got["mean"], m)
    assert np.array_equal(got["steps"], st)


def test_record_layout_single_process_roundtrip():
    """RecordLayout with one rank: the root buffer is the rank buffer (the ekya_gather_decisions
    one-rank path copies it), and unpack returns the rows written, for any chunk count."""
    V = 10
    for total, n_chunks in ((0, 8), (1, 8), (37, 8), (64, 4), (65, 1)):
        L = shard.RecordLayout(total, 1, V, n_chunks)
        buf = torch.zeros(L.rank_bytes, dtype=torch.uint8)
        for c in range(L.n_chunks):
            b0, b1 = L.chunk_range(0, c)
            v = L.views(buf, 0, c)
            v["sum"][:] = torch.arange(b0, b1, dtype=torch.int64).to(torch.uint64)
            v["alloc"][:] = torch.arange(b0, b1, dtype=torch.int32).to(torch.uint16)[:, None]
        got = L.unpack(buf.clone())
        if total:
            assert got["sum"].to(torch.int64).tolist() == list(range(total))
            assert (got["alloc"].to(torch.int32) == torch.arange(total)[:, None]).all()


def test_shard_ranges_partition():
    for total in (0, 1, 7, 65536, 1000000):
        for P in (1, 2, 3, 4, 8):
            rs = [shard.shard_range(total, P, r) for r in range(P)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c and a <= b


def test_shard_generation_is_rank_independent():
    """A rank's shard generated alone equals the same rows of the full batch."""
    cfg = synth.SchedConfig(**{**synth.CONFIG2.__dict__, "n_inst": 10})
    full = synth.sched_tables(cfg)
    part = synth.sched_tables(cfg, 6, 10)
    for k in full:
        assert torch.equal(full[k][6:10], part[k])
    rows_full = synth.list_allocs(cfg, 5)
    rows_part = synth.list_allocs(cfg, 5, 6, 10)
    assert torch.equal(rows_full[6:10], rows_part)
    pc = synth.ProfileConfig("p", 9, 40, 27, 18)
    pf, pp = synth.profile_inputs(pc), synth.profile_inputs(pc, 4, 9)
    for k in pf:
        assert torch.equal(pf[k][4:9], pp[k])
