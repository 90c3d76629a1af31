"""Basis build of configs[1]: wall time of build_coarse_basis and subspace-iteration counts."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402

spec = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1_mbb_1024x512"]
m = Msfem.from_spec(spec)
m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m.build_coarse_basis()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    phi, nk, lam = m.get_basis()
    print(f"basis {dt * 1e3:.1f} ms, classes {m.info()['n_classes']}, max subspace iterations "
          f"{m.info()['eig_iters']}")
