"""Times the per-design-iteration setup of a config on the GPU: filter/project, spectral
basis, coarse assembly (Galerkin cell products + factorisation), and one PCG solve.
usage: python scripts/time_setup.py [config ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402

for name in sys.argv[1:] or ["c4_mbb_5120x2560", "c3_square_2048"]:
    spec = W.CONFIGS[name]
    m = Msfem.from_spec(spec)
    x = torch.as_tensor(W.design_tile(spec), device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for rep in range(2):
        ev[0].record(m.stream)
        m.filter_project(x)
        ev[1].record(m.stream)
        m.build_coarse_basis()
        ev[2].record(m.stream)
        m.assemble_coarse()
        ev[3].record(m.stream)
        its, comps, nc = m.pcg_solve(tol=spec.tol, max_it=20000)
        ev[4].record(m.stream)
        torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    kb = m.bench_kernels(reps=3)
    print(f"{name}: filter {t[0]:.2f} ms, basis {t[1]:.2f} ms, assemble {t[2]:.2f} ms "
          f"(galerkin {kb['assemble_local'][0]:.2f}?), pcg {t[3]:.1f} ms iters {its}; "
          f"workspace {m.info()['workspace_bytes'] / 2**30:.2f} GiB", flush=True)
    m.close()
    del m
    torch.cuda.empty_cache()
