import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1411_3923_b200 import Msfem
from oracle import problem
base = W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary",
                    n_modes=16, seed=41, lam_threshold=5e-3)
x = W.design_tile(base)
for Emin in (1e-3,):
    spec = base.replace(Emin=Emin)
    m = Msfem.from_spec(spec)
    m.filter_project(torch.as_tensor(x, device="cuda"))
    m.build_coarse_basis()
    _, nk, lam = m.get_basis()
    print("nkept", np.bincount(nk))
    m.assemble_coarse()
    it, comps, nc = m.pcg_solve(tol=1e-8)
    print(os.environ.get("TAG"), "iters", it, comps, nc, flush=True)
