"""Times pcg_solve alone (CUDA events, 5 repeats after a warm-up) on one config: the PCG
driver's share of a step, used to A/B the run-time switches of the iteration loop."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from paper_1411_3923_b200 import Msfem

name = sys.argv[1] if len(sys.argv) > 1 else "c1_mbb_1024x512"
spec = W.CONFIGS[name]
m = Msfem.from_spec(spec)
x = torch.as_tensor(W.design_tile(spec), device="cuda")
m.filter_project(x)
m.build_coarse_basis()
m.assemble_coarse()
m.pcg_solve(tol=spec.tol, max_it=20000)
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    its, comps, nc = m.pcg_solve(tol=spec.tol, max_it=20000)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps(dict(config=name, env={k: v for k, v in os.environ.items() if k.startswith("MSF_")},
                      iters=its, pcg_ms=sorted(ts), us_per_iter=min(ts) * 1e3 / max(its))))
