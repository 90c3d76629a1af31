"""Worker of tests/test_gpu_nccl_multi.py: run under torch.distributed.run with one process per
GPU.  Every rank solves its strip of a small robust problem through the NCCL transport (halo
send/recv, all-reduces, the captured per-iteration graphs) and also the whole problem on its own
GPU; it checks iteration counts (+-1), compliances and its owned displacement columns against
the single-GPU solve, then the robust sensitivities.  Exits non-zero on any mismatch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1411_3923_b200 as pkg  # noqa: E402
import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402


def main():
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    specs = [
        # strips of 16 node columns at 2 ranks: 8-column halos, streaming sweep
        W.small_spec(nelx=32 * ws // 2, nely=16, cx=8, cy=8, tile=(8, 8), rmin=2.5, beta=8.0,
                     etas=(0.7, 0.5, 0.3), dilated=2, bc="mbb", seed=23, Emin=1e-6),
        # strips of 3-6 columns: one-column halos, colour-phase sweep
        W.small_spec(nelx=6 * ws, nely=12, cx=3, cy=3, seed=41, Emin=1e-6),
    ]
    for spec in specs:
        x = W.design_tile(spec)
        fx, f = W.fixed_mask(spec), W.load_vector(spec)
        uid = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        m = Msfem(pkg.problem_from_spec(spec), fx, f, device=dev, rank=rank, nranks=ws,
                  transport=pkg.MSF_TRANSPORT_NCCL, handle=uid[0])
        s = Msfem.from_spec(spec, device=dev)
        xd = torch.as_tensor(x, device=dev)
        for ctx in (m, s):
            ctx.filter_project(xd)
            ctx.build_coarse_basis()
            ctx.assemble_coarse()
        nny = spec.nely + 1
        b = pkg.strip_bounds(pkg.problem_from_spec(spec), rank, ws)
        ul = torch.zeros(spec.n_rhs, b["ncols"] * nny * 2, dtype=torch.float64, device=dev)
        ug = torch.zeros(spec.n_rhs, spec.n_dof, dtype=torch.float64, device=dev)
        its_m, comp_m, nc_m = m.pcg_solve(tol=1e-10, u=ul)
        its_s, comp_s, nc_s = s.pcg_solve(tol=1e-10, u=ug)
        assert not nc_m and not nc_s
        for k in range(spec.n_rhs):
            assert abs(its_m[k] - its_s[k]) <= 1, (spec.name, its_m, its_s)
            assert abs(comp_m[k] - comp_s[k]) <= 1e-9 * abs(comp_s[k]), (spec.name, comp_m, comp_s)
        o0, o1 = b["own0"] - b["gox"], b["own1"] - b["gox"]
        mine = ul.view(spec.n_rhs, b["ncols"], nny, 2)[:, o0:o1].cpu().numpy()
        ref = ug.view(spec.n_rhs, spec.nelx + 1, nny, 2)[:, b["own0"]:b["own1"]].cpu().numpy()
        for k in range(spec.n_rhs):
            assert np.abs(mine[k] - ref[k]).max() <= 1e-8 * np.abs(ref[k]).max(), (spec.name, rank, k)
        nt = spec.tile_x * spec.tile_y
        dFm, dgm = (torch.empty(nt, dtype=torch.float64, device=dev) for _ in range(2))
        dFs, dgs = (torch.empty(nt, dtype=torch.float64, device=dev) for _ in range(2))
        Fm, gm, _ = m.sensitivities(kappa=1.0, volfrac=0.5, dF=dFm, dg=dgm)
        Fs, gs, _ = s.sensitivities(kappa=1.0, volfrac=0.5, dF=dFs, dg=dgs)
        assert abs(Fm - Fs) <= 1e-8 * abs(Fs) and abs(gm - gs) <= 1e-12
        assert float((dFm - dFs).abs().max()) <= 1e-7 * float(dFs.abs().max())
        m.close()
        s.close()
        dist.barrier()
        if rank == 0:
            print(f"nccl strips ok: {spec.name} on {ws} ranks, iterations {its_m} (single GPU {its_s})", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
