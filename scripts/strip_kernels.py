"""msf_bench_kernels of one rank of an N-strip partition of configs[4] (in-process group)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1411_3923_b200 import MsfemGroup
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
spec = W.CONFIGS["c4_mbb_5120x2560"]
x = torch.as_tensor(W.design_tile(spec), device="cuda")
g = MsfemGroup.from_spec(spec, N)
g.filter_project(x)
g.build_coarse_basis()
g.assemble_coarse()
for r in (0, N // 2):
    for nr in ("1", "3"):
        os.environ["MSF_BENCH_NR"] = nr
        kb = g.ranks[r].bench_kernels(reps=20)
        print("rank", r, "nr", nr, json.dumps({k: round(v[0], 4) for k, v in kb.items() if v[0] > 0}), flush=True)
