"""Debug: nested-dissection coarse solve vs a dense solve of the gathered K_c blocks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_1411_3923_b200 import Msfem

def dense_kc(m, spec, rhs):
    D, U = m.get_coarse_blocks(rhs)
    nb, mc = D.shape[0], D.shape[1]
    K = np.zeros((nb * mc, nb * mc))
    for i in range(nb):
        K[i*mc:(i+1)*mc, i*mc:(i+1)*mc] = D[i]
        if i + 1 < nb:
            K[i*mc:(i+1)*mc, (i+1)*mc:(i+2)*mc] = U[i]
            K[(i+1)*mc:(i+2)*mc, i*mc:(i+1)*mc] = U[i].T
    return K

for name, spec in [
    ("u128x64", W.small_spec(nelx=128, nely=64, cx=4, cy=4, Emin=1.0, E0=2.0, design="iid")),
    ("iid128x64", W.small_spec(nelx=128, nely=64, cx=4, cy=4, Emin=1e-9)),
    ("k5_36x20", W.small_spec(nelx=36, nely=20, cx=4, cy=4, n_modes=5, tile=(12, 10), Emin=1e-6)),
    ("thr64x32", W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary",
                              n_modes=16, seed=41, lam_threshold=5e-3, Emin=1e-3)),
    ("thr64x32_1e-6", W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary",
                              n_modes=16, seed=41, lam_threshold=5e-3, Emin=1e-6)),
    ("thr64x32_1e-9", W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary",
                              n_modes=16, seed=41, lam_threshold=5e-3, Emin=1e-9)),
    ("k16_64x32", W.small_spec(nelx=64, nely=32, cx=8, cy=8, tile=(32, 16), design="binary",
                              n_modes=16, seed=41, Emin=1e-3)),
    ("k8_64x32", W.small_spec(nelx=64, nely=32, cx=8, cy=8, n_modes=8, seed=41, Emin=1e-3)),
]:
    m = Msfem.from_spec(spec)
    m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
    m.build_coarse_basis()
    try:
        m.assemble_coarse()
        rng = np.random.default_rng(0)
        for rhs in range(len(spec.etas)):
            K = dense_kc(m, spec, rhs)
            n = K.shape[0]
            b = rng.standard_normal(n)
            x = m.coarse_solve(rhs, torch.as_tensor(b, device="cuda")).cpu().numpy() if False else None
            bd = torch.as_tensor(b, device="cuda")
            xd = torch.empty_like(bd)
            m.coarse_solve(rhs, bd, xd)
            x = xd.cpu().numpy()
            xr = np.linalg.solve(K, b)
            print(name, rhs, "n", n, "cond", np.linalg.cond(K), "rel err", np.linalg.norm(x - xr) / np.linalg.norm(xr),
                  "resid", np.linalg.norm(K @ x - b) / np.linalg.norm(b), flush=True)
    except Exception as e:
        print(name, "ERROR", e, flush=True)
    m.close()
