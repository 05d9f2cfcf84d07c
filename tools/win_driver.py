"""Run the NEXT-1 window timeline once over config-4 instances (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2012_10557_b200 import ekya  # noqa: E402

B = int(os.environ.get("KB_B", 65536))
cfg = synth.SchedConfig(**{**synth.CONFIG4.__dict__, "n_inst": B})
torch.cuda.set_device(0)
h = ekya.Handle(0)
T = synth.sched_tables(cfg, 0, B, device="cuda")
for _ in range(2):
    ekya.window_schedule(h, T, cfg.units, cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)
torch.cuda.synchronize()
assert h.last_error() == 0
