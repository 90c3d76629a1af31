"""msf_bench_kernels table (ms per launch-set, HBM fraction) of a config at 1 and all realisations."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1411_3923_b200 import Msfem
name = sys.argv[1] if len(sys.argv) > 1 else "c4_mbb_5120x2560"
spec = W.CONFIGS[name]
m = Msfem.from_spec(spec)
m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
m.build_coarse_basis()
m.assemble_coarse()
for nr in ("1", str(spec.n_rhs)):
    os.environ["MSF_BENCH_NR"] = nr
    kb = m.bench_kernels(reps=10)
    print(os.environ.get("TAG", ""), "nr", nr, json.dumps({k: round(v[0], 4) for k, v in kb.items() if v[0] > 0}), flush=True)
