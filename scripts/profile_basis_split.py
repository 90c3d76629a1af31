"""Basis build time of configs[1] with the subspace-iteration cap at 1 (factorisation + one
iteration) and at the default (60, converges in ~16)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem, problem_from_spec  # noqa: E402

spec = W.CONFIGS["c1_mbb_1024x512"]
for cap in (1, 2, 0):
    p = problem_from_spec(spec)
    p.eig_max_iter = cap
    m = Msfem(p, W.fixed_mask(spec), W.load_vector(spec))
    m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m.build_coarse_basis()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"cap {cap}: {dt * 1e3:.1f} ms")
