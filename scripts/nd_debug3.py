import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import workloads as W
from paper_1411_3923_b200 import Msfem
from oracle import problem
from test_gpu_parity import ctx_for
base = W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary",
                    n_modes=16, seed=41, lam_threshold=5e-3)
x = W.design_tile(base)
fx, f = W.fixed_mask(base), W.load_vector(base)
for variant in range(4):
    spec = base.replace(Emin=1e-3)
    m, _ = ctx_for(spec, x)
    m.build_coarse_basis()
    _, nk, lam = m.get_basis()
    m.assemble_coarse()
    if variant == 1:
        ref = problem.solve(spec, x, fx, f, tol=1e-8)
        print("ref", ref["iters"])
    if variant == 2:
        torch.cuda.synchronize()
    it, comps, nc = m.pcg_solve(tol=1e-8)
    print(variant, "iters", it, comps, flush=True)
