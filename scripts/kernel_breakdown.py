"""Per-kernel times of one PCG iteration (msf_bench_kernels) at 1 and all active realisations
for a BASELINE config (default configs[1]); prints a table of ms per launch-set."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c1_mbb_1024x512"
    spec = W.CONFIGS[name]
    m = Msfem.from_spec(spec)
    m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
    m.build_coarse_basis()
    m.assemble_coarse()
    m.pcg_solve(tol=spec.tol, max_it=20000)
    rows = {}
    for nr in (1, spec.n_rhs):
        os.environ["MSF_BENCH_NR"] = str(nr)
        rows[nr] = m.bench_kernels(reps=50)
    print(f"{name}: ms per launch-set (sgs_colour = one symmetric sweep of 7 launches)")
    print("| kernel | 1 realisation | %d realisations |" % spec.n_rhs)
    print("|---|---|---|")
    for k in rows[1]:
        print(f"| {k} | {rows[1][k][0]:.4f} | {rows[spec.n_rhs][k][0]:.4f} |")


if __name__ == "__main__":
    main()
