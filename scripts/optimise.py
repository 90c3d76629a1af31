"""Robust topology optimisation with the library: N design iterations of a BASELINE config
(default configs[1]) with the design evolving (filter -> projections -> basis -> K_c -> PCG
x 3 realisations -> robust sensitivities -> OC), one JSON line per iteration: robust
objective F = E[c] + kappa sqrt(Var c), volume constraint g, per-realisation PCG iterations
and compliances, wall time of the iteration.
usage: python scripts/optimise.py [config] [iterations]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1_mbb_1024x512"
    n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    spec = W.CONFIGS[name]
    m = Msfem.from_spec(spec)
    # start from the uniform design at the volume fraction (the usual topology-optimisation start)
    x = torch.full((spec.tile_x * spec.tile_y,), spec.volfrac, dtype=torch.float64, device="cuda")
    xn = torch.empty_like(x)
    for it in range(n_it):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        its, comps, F, g = m.design_iteration(x, xn, tol=spec.tol, max_it=20000, kappa=spec.kappa,
                                              volfrac=spec.volfrac)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        change = float((xn - x).abs().max())
        print(json.dumps(dict(iteration=it, F=F, g=g, pcg_iters=its, compliances=comps,
                              max_change=change, seconds=round(dt, 4))), flush=True)
        x.copy_(xn)


if __name__ == "__main__":
    main()
