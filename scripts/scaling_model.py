"""Strip-partition scaling model for BASELINE configs[4] (5120x2560 MBB, 26.2M DOF) from
single-GPU MEASUREMENTS (this box has one GPU):

* the full problem: PCG iteration counts per realisation, coarse-solve time per iteration
  at 1 and 3 active realisations (replicated on every rank), coarse assembly time;
* strip-sized problems (nelx = 5120/N, same rows, coarse cells and design): the fine-grid
  kernels of one PCG iteration (apply, 2 SGS sweeps, residual, restriction, prolongation,
  update + F0, p update) at 1 and 3 active realisations;
* ASSUMED: t_comm per NCCL operation over NVLink (argument, default 8 us); 14 halo exchanges +
  4 all-reduces per iteration.

T_iter(N, k) = fine(5120/N, k) + coarse(k) + [N > 1] * 18 * t_comm ;  the step time sums over
the iterations with k active realisations, plus the replicated assembly.  Prints a markdown
table."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem  # noqa: E402

FINE = ["apply", "restrict", "prolong", "residual", "update_f0", "p_update"]


def kernels(m, nr):
    os.environ["MSF_BENCH_NR"] = str(nr)
    kb = m.bench_kernels(reps=10)
    fine = sum(kb[k][0] for k in FINE) + 2 * kb["sgs_colour"][0]
    return fine, kb["coarse_solve"][0], kb


def setup(spec):
    m = Msfem.from_spec(spec)
    x = torch.as_tensor(W.design_tile(spec), device="cuda")
    m.filter_project(x)
    m.build_coarse_basis()
    torch.cuda.synchronize()
    t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t[0].record()
    m.assemble_coarse()
    t[1].record()
    torch.cuda.synchronize()
    return m, t[0].elapsed_time(t[1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t-comm-us", type=float, default=8.0)
    a = ap.parse_args()
    spec = W.CONFIGS["c4_mbb_5120x2560"]
    m, assemble_ms = setup(spec)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    its, comps, _ = m.pcg_solve(tol=spec.tol, max_it=20000)
    t1.record()
    torch.cuda.synchronize()
    pcg_ms = t0.elapsed_time(t1)
    _, coarse1, kb1 = kernels(m, 1)
    _, coarse3, kb3 = kernels(m, 3)
    del m
    torch.cuda.empty_cache()
    its_sorted = sorted(its, reverse=True)            # iterations with >=1, >=2, 3 active
    n_k = {1: its_sorted[0] - its_sorted[1], 2: its_sorted[1] - its_sorted[2], 3: its_sorted[2]}
    rows = []
    for N in (1, 2, 4, 8):
        sub = spec.replace(name=f"c4_strip_{N}", nelx=spec.nelx // N)
        ms, _ = setup(sub)
        f1, _, _ = kernels(ms, 1)
        f3, _, _ = kernels(ms, 3)
        del ms
        torch.cuda.empty_cache()
        f2 = (f1 + f3) / 2
        comm = 0.0 if N == 1 else 18 * a.t_comm_us * 1e-3
        it_ms = {1: f1 + coarse1 + comm, 2: f2 + (coarse1 + coarse3) / 2 + comm, 3: f3 + coarse3 + comm}
        pcg = sum(n_k[k] * it_ms[k] for k in (1, 2, 3))
        rows.append(dict(N=N, fine1=f1, fine3=f3, iter1=it_ms[1], pcg_ms=pcg,
                         step_ms=pcg + assemble_ms))
    base = rows[0]["step_ms"]
    print(json.dumps(dict(iters=its, pcg_ms_measured=pcg_ms, assemble_ms=assemble_ms,
                          coarse1_ms=coarse1, coarse3_ms=coarse3, t_comm_us=a.t_comm_us)))
    print("| N | fine grid / iteration (1 real., ms) | coarse (1 real., ms) | comm (ms) | "
          "iteration (1 real., ms) | PCG per design iteration (s) | + assembly (s) | speedup |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        comm = 0.0 if r["N"] == 1 else 18 * a.t_comm_us * 1e-3
        print(f"| {r['N']} | {r['fine1']:.3f} | {coarse1:.3f} | {comm:.3f} | {r['iter1']:.3f} | "
              f"{r['pcg_ms'] / 1e3:.2f} | {r['step_ms'] / 1e3:.2f} | {base / r['step_ms']:.2f} |")


if __name__ == "__main__":
    main()
