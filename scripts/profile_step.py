"""One design iteration of a BASELINE config for profiling (ncu): setup + one warm step,
then `--steps` more.  Prints the PCG iteration counts.  Not a benchmark (use bench.py)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1_mbb_1024x512")
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    spec = W.CONFIGS[a.config]
    m = Msfem.from_spec(spec)
    x = torch.as_tensor(W.design_tile(spec), device="cuda")
    xn = torch.empty_like(x)
    for _ in range(1 + a.steps):
        its, comps, F, g = m.design_iteration(x, xn, tol=spec.tol, max_it=5000)
    torch.cuda.synchronize()
    print("iters", its, "launches per PCG iteration", m.info()["pcg_iter_launches"])


if __name__ == "__main__":
    main()
