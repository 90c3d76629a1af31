"""Runs msf_bench_kernels once on a BASELINE config so that `ncu -k regex:<kernel>` can
capture launches of any path kernel in its PCG launch configuration.
usage: ncu ... python scripts/profile_kernel.py [config] [n_active_realisations]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4_mbb_5120x2560"
os.environ["MSF_BENCH_NR"] = sys.argv[2] if len(sys.argv) > 2 else "1"
spec = W.CONFIGS[name]
m = Msfem.from_spec(spec)
m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
m.build_coarse_basis()
m.assemble_coarse()
kb = m.bench_kernels(reps=3)
print({k: round(v[0], 4) for k, v in kb.items()})
