"""Rounding sensitivity of the PCG iteration count (tests/test_gpu_strips.py bars).

The eroded realisation of the robust_32x16 test problem needs ~137 preconditioned CG
iterations on 1,122 DOF: far past the point where finite-precision CG has lost
orthogonality, so its iteration count is chaotic under rounding.  This script perturbs the
design tile by 1e-15 (relative, seeded) and histograms the iteration count of the single-GPU
path (40 seeds) and of two strips (12 seeds); seed 0 is the unperturbed tile.  Output:
profiles/r01_rounding_spread.txt."""
import collections
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem, MsfemGroup  # noqa: E402
from test_gpu_parity import SPECS  # noqa: E402


def main():
    spec = SPECS["robust_32x16"]
    x0 = W.design_tile(spec)
    hs, hg = collections.Counter(), collections.Counter()
    for seed in range(40):
        rng = np.random.default_rng(seed)
        xp = x0 * (1 + 1e-15 * rng.standard_normal(x0.size)) if seed else x0
        x = torch.as_tensor(xp, device="cuda")
        m = Msfem.from_spec(spec)
        m.filter_project(x)
        m.build_coarse_basis()
        m.assemble_coarse()
        hs[m.pcg_solve(tol=1e-8)[0][0]] += 1
        m.close()
        if seed < 12:
            g = MsfemGroup.from_spec(spec, 2)
            g.filter_project(x)
            g.build_coarse_basis()
            g.assemble_coarse()
            hg[g.pcg_solve(tol=1e-8)[0][0]] += 1
            g.close()
    print("robust_32x16 eroded realisation, design tile perturbed by 1e-15 (relative):")
    print("  single GPU, 40 seeds: iterations", dict(sorted(hs.items())))
    print("  2 strips,   12 seeds: iterations", dict(sorted(hg.items())))


if __name__ == "__main__":
    main()
