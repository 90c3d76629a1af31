"""Strip-partition scaling model for BASELINE configs[4] (5120x2560 MBB, 26.2M DOF) from
single-GPU MEASUREMENTS (this pool has one GPU per box):

* the full problem on one GPU: PCG iteration counts per realisation, PCG time, the
  replicated per-design-iteration setup (filter + projection + spectral basis) and the K_c
  assembly;
* the strip partition over N = 2, 4, 8 ranks, all ranks as contexts of one process on the
  one GPU (MSF_TRANSPORT_GROUP): every rank's own kernels, timed by msf_bench_kernels on that
  rank's context in the PCG launch configuration at 1 and 3 active realisations: the
  fine-grid kernels of one PCG iteration on its wide-halo strip (apply, pre-smoothing sweep
  with the residual update, residual, restriction, prolongation, post-smoothing sweep,
  direction / solution update), its share of the coarse solve (forward and back over its box
  of the nested dissection, the replicated interface fronts) and of the assembly (Galerkin
  products + box factorisation, the replicated interface factorisation).  A step takes the
  slowest rank;
* ASSUMED (not measurable on one GPU): t_comm per NCCL operation over NVLink (default 8 us);
  4 halo exchanges + 4 all-reduces per PCG iteration (wide-halo strips); the
  all-reduce of the interface fronts at assembly at --allreduce-gbps (default 300).

T_iter(N, k) = max_r [fine_r(k) + coarse_r(k)] + [N > 1] 8 t_comm ;  the step sums over the
iterations with k active realisations, plus setup + assembly.  Prints a markdown table."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_1411_3923_b200 import Msfem, MsfemGroup  # noqa: E402

FINE = ["apply", "sgs_pre_update", "residual", "restrict", "prolong", "sgs_sweep", "p_update"]
N_COMM = 8   # NCCL operations per PCG iteration: halos q, z, t, z + all-reduces p.q, |r|^2, interface rhs, r.z
COARSE = ["coarse_fwd_local", "coarse_top", "coarse_back_local"]


def rank_times(m, nr, reps):
    os.environ["MSF_BENCH_NR"] = str(nr)
    kb = m.bench_kernels(reps=reps)
    fine = sum(kb[k][0] for k in FINE)
    coarse = sum(kb[k][0] for k in COARSE)
    return fine, coarse, kb["assemble_local"][0], kb["assemble_top"][0]


def timed(fn):
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0.record()
    out = fn()
    t1.record()
    torch.cuda.synchronize()
    return out, t0.elapsed_time(t1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--t-comm-us", type=float, default=8.0)
    ap.add_argument("--allreduce-gbps", type=float, default=300.0)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    spec = W.CONFIGS["c4_mbb_5120x2560"]
    x = torch.as_tensor(W.design_tile(spec), device="cuda")

    m = Msfem.from_spec(spec)
    _, setup_ms = timed(lambda: (m.filter_project(x), m.build_coarse_basis()))
    _, assemble_ms = timed(m.assemble_coarse)
    (its, comps, _), pcg_ms = timed(lambda: m.pcg_solve(tol=spec.tol, max_it=20000))
    f1, c1, al1, at1 = rank_times(m, 1, a.reps)
    f3, c3, _, _ = rank_times(m, 3, a.reps)
    mc = m.info()["m"]
    del m
    torch.cuda.empty_cache()
    its_sorted = sorted(its, reverse=True)            # iterations with >=1, >=2, 3 active
    n_k = {1: its_sorted[0] - its_sorted[1], 2: its_sorted[1] - its_sorted[2], 3: its_sorted[2]}

    rows = [dict(N=1, fine1=f1, coarse1=c1, fine3=f3, coarse3=c3, comm=0.0,
                 assemble=al1 + at1, allreduce=0.0)]
    for N in (2, 4, 8):
        g = MsfemGroup.from_spec(spec, N)
        g.filter_project(x)
        g.build_coarse_basis()
        g.assemble_coarse()
        per = [(rank_times(r, 1, a.reps), rank_times(r, 3, a.reps)) for r in g.ranks]
        g.close()
        del g
        torch.cuda.empty_cache()
        worst1 = max(per, key=lambda t: t[0][0] + t[0][1])[0]
        worst3 = max(per, key=lambda t: t[1][0] + t[1][1])[1]
        asm = max(t[0][2] for t in per) + max(t[0][3] for t in per)
        ar_bytes = spec.n_rhs * (2 * N + 1) * mc * mc * 8
        rows.append(dict(N=N, fine1=worst1[0], coarse1=worst1[1], fine3=worst3[0],
                         coarse3=worst3[1], comm=N_COMM * a.t_comm_us * 1e-3, assemble=asm,
                         allreduce=ar_bytes / (a.allreduce_gbps * 1e9) * 1e3))
    for r in rows:
        it1 = r["fine1"] + r["coarse1"] + r["comm"]
        it3 = r["fine3"] + r["coarse3"] + r["comm"]
        r["iter1"] = it1
        r["pcg_ms"] = n_k[1] * it1 + n_k[2] * (it1 + it3) / 2 + n_k[3] * it3
        r["step_ms"] = r["pcg_ms"] + setup_ms + r["assemble"] + r["allreduce"]
    base = rows[0]["step_ms"]
    print(json.dumps(dict(iters=its, pcg_ms_measured=pcg_ms, setup_ms=setup_ms,
                          assemble_ms_measured=assemble_ms, t_comm_us=a.t_comm_us,
                          allreduce_gbps=a.allreduce_gbps, m=mc)))
    print("| N | fine grid / iter (1 real., ms) | coarse / iter (1 real., ms) | comm / iter (ms) | "
          "iteration (1 real., ms) | PCG (s) | assembly + all-reduce (s) | setup (s) | step (s) | speedup |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['N']} | {r['fine1']:.3f} | {r['coarse1']:.3f} | {r['comm']:.3f} | {r['iter1']:.3f} | "
              f"{r['pcg_ms'] / 1e3:.2f} | {(r['assemble'] + r['allreduce']) / 1e3:.3f} | {setup_ms / 1e3:.3f} | "
              f"{r['step_ms'] / 1e3:.2f} | {base / r['step_ms']:.2f} |")


if __name__ == "__main__":
    main()
