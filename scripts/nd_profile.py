"""Coarse solve of configs[4] (or argv[1]) for a launch-list / ncu capture: setup, basis,
assembly, then 3 coarse solves of all realisations and 3 of one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1411_3923_b200 import Msfem
name = sys.argv[1] if len(sys.argv) > 1 else "c4_mbb_5120x2560"
spec = W.CONFIGS[name]
m = Msfem.from_spec(spec)
m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
m.build_coarse_basis()
m.assemble_coarse()
inf = m.info()
n = inf["coarse_slots"]
b = torch.as_tensor(np.random.default_rng(0).standard_normal(n), device="cuda")
x = torch.empty_like(b)
for _ in range(3):
    m.coarse_solve(0, b, x)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(m.stream)
for _ in range(10):
    m.coarse_solve(0, b, x)
ev[1].record(m.stream)
torch.cuda.synchronize()
print("coarse_solve (1 rhs, incl. 2 copies) ms", ev[0].elapsed_time(ev[1]) / 10)
