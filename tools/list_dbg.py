import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth, numpy as np
from paper_2012_10557_b200 import ekya
B = int(sys.argv[1]); N = int(sys.argv[2])
cfg = synth.SchedConfig(**{**synth.CONFIG4.__dict__, "n_inst": B})
h = ekya.Handle(0)
Td = synth.sched_tables(cfg, device="cuda")
rows = synth.list_allocs(cfg, N, 0, B, device="cuda")
ls, lm, lc = ekya.eval_list(h, Td, rows, cfg.units, cfg.steal_units, cfg.unit_gpu_seconds, cfg.a_min)
print("B", B, "N", N, "err", h.last_error())
