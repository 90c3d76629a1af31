import torch, workloads as W
from paper_1411_3923_b200 import Msfem
s = W.small_spec(nelx=16, nely=8, cx=4, cy=4, seed=21)
m = Msfem.from_spec(s)
m.filter_project(torch.as_tensor(W.design_tile(s), device="cuda"))
m.build_coarse_basis(); m.assemble_coarse()
try:
    print(m.pcg_solve(tol=1e-8))
except Exception as e:
    print("ERR", e)
