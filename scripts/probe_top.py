"""Debug probe: GPU coarse solve vs numpy dense solve on the threshold-mode case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1411_3923_b200 import Msfem
base = W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary", n_modes=16, seed=41, lam_threshold=5e-3)
x = W.design_tile(base)
for Emin in (1e-3, 1e-6, 1e-9):
    s = base.replace(Emin=Emin)
    m = Msfem.from_spec(s)
    m.filter_project(torch.as_tensor(x, device="cuda")); m.build_coarse_basis(); m.assemble_coarse()
    inf = m.info(); nb, mm = inf["ncx"] + 1, inf["m"]
    D, U = m.get_coarse_blocks(0)
    Kc = np.zeros((nb * mm, nb * mm))
    for I in range(nb):
        Kc[I*mm:(I+1)*mm, I*mm:(I+1)*mm] = D[I]
        if I + 1 < nb:
            Kc[I*mm:(I+1)*mm, (I+1)*mm:(I+2)*mm] = U[I]; Kc[(I+1)*mm:(I+2)*mm, I*mm:(I+1)*mm] = U[I].T
    b = np.random.default_rng(0).standard_normal(nb * mm)
    c = torch.empty(nb * mm, dtype=torch.float64, device="cuda")
    m.coarse_solve(0, torch.as_tensor(b, device="cuda"), c); torch.cuda.synchronize()
    ref = np.linalg.solve(Kc, b)
    ev = np.linalg.eigvalsh(Kc)
    print(Emin, "cond", ev.max() / ev.min(), "min eig", ev.min(), "rel err", np.linalg.norm(c.cpu().numpy() - ref) / np.linalg.norm(ref),
          "pcg", m.pcg_solve(tol=1e-8)[0], flush=True)
