"""Filter + basis + coarse assembly of one BASELINE config (for an ncu launch list of the
assembly kernels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402

spec = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4_mbb_5120x2560"]
m = Msfem.from_spec(spec)
m.filter_project(torch.as_tensor(W.design_tile(spec), device="cuda"))
m.build_coarse_basis()
m.assemble_coarse()
torch.cuda.synchronize()
print("ok")
