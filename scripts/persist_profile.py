"""Debug: phase timeline of the persistent PCG kernel on the bench workload (1 and 3 rhs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["MSF_PERSIST_PROFILE"] = "1"
import torch
import workloads as W
from paper_1411_3923_b200 import Msfem
s = W.CONFIGS["c1_mbb_1024x512"]
m = Msfem.from_spec(s)
m.filter_project(torch.as_tensor(W.design_tile(s), device="cuda"))
m.build_coarse_basis(); m.assemble_coarse()
for nr in (3, 1):
    its, comps, _ = m.pcg_solve(n_rhs=nr, tol=1e-8)
    print(nr, its, flush=True)
