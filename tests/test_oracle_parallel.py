"""The oracle's host thread pool (oracle.per_instance_parallel) is marshalling only: over
independent instances it must reproduce the single-threaded oracle bit for bit, including
per-instance array arguments (LIST rows) sliced with their instance block."""
import numpy as np

import oracle
import synth


def _inst(cfg, n):
    c = synth.SchedConfig(**{**cfg.__dict__, "n_inst": n})
    T = synth.sched_tables(c)
    return c, oracle.Instances(*(T[k].numpy() for k in ("stale", "cost", "post", "lam_min_units", "lam_factor")),
                               c.units, c.steal_units, c.unit_gpu_seconds, c.a_min)


def test_parallel_equals_serial():
    c, inst = _inst(synth.CONFIG2, 37)
    rows = synth.list_allocs(c, 64).numpy()
    for fn, args in ((oracle.eval_list, (rows,)), (oracle.thief, (oracle.STEEPEST,)),
                     (oracle.thief, (oracle.LITERAL,)), (oracle.eval_grid, ())):
        a = fn(inst, *args)
        b = oracle.per_instance_parallel(fn, inst, *args, threads=5)
        assert len(a) == len(b)
        for x, y in zip(a, b):
            if isinstance(x, np.ndarray):
                assert x.dtype == y.dtype and np.array_equal(x, y)
            else:
                assert x == y
