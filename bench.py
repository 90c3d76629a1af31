"""Benchmark of the B200 MsFEM-PCG hot path (BASELINE.json metric).

A *step* is one pass of the whole hot path over the configs[4] workload
(MBB 5120x2560, 26,229,762 DOF, the paper's largest size, PAPER.md l.439 -- the config the
BASELINE metric is quoted on, and it fits one B200):
filter_project (3 Heaviside realisations) -> build_coarse_basis (dilated realisation) ->
assemble_coarse (3 Galerkin K_c + factorisations) -> pcg_solve (3 realisations, tol 1e-8,
x0 = 0) -> sensitivities -> oc_update, always from the same seeded design tile, so every
step does identical work.  metric = sum over realisations of PCG iterations x n_dof per
second (whole job, all ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): the grid of the SAME workload is strip-partitioned over the ranks
(msf_dist_setup with the NCCL transport; halo exchanges and all-reduces
inside the library, K_c distributed by block chains with a replicated interface system), so
the total work is fixed (strong scaling);
value = n_dof x PCG iterations / max-over-ranks time.  --mode replicas instead runs an
independent copy per rank (weak scaling).  After the timed region a one-GPU run also
records the configs[3] contrast sweep (E_min 1e-3 / 1e-6 / 1e-9: PCG iterations and
DOF*iter/s per contrast).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "PCG DOF*iterations/s (matvec+2-level precond), 3 robust realisations"
UNIT = "DOF*iter/s"
DEFAULT_CONFIG = "c4_mbb_5120x2560"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def hbm_peak():
    try:
        with open(PEAKS) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample_spec(spec, cells=(8, 4)):
    """Bounded sample of the same workload for the oracle: the recipe (tile, filter,
    projection, 3 realisations, coarse cells, modes, tolerance) on a sub-grid of 8 x 4 coarse
    cells (configs[4]: 160x80 elements; about 10-30 s of oracle work).  The reference arm
    times every one of its warm-up + timed steps, so it uses 4 x 2 cells (80x40, a few s)."""
    nx, ny = cells[0] * spec.cx, cells[1] * spec.cy
    nx += (-nx) % spec.tile_x
    ny += (-ny) % spec.tile_y
    return spec.replace(name=f"{spec.name}_cpu_sample_{nx}x{ny}", nelx=nx, nely=ny)


def oracle_sample(spec, cells=(8, 4)):
    """Times the oracle (as it stands) on the bounded sample; returns (value, seconds, iters)."""
    from oracle import problem
    s = cpu_sample_spec(spec, cells)
    x = W.design_tile(s)
    fx, f = W.fixed_mask(s), W.load_vector(s)
    t0 = time.perf_counter()
    out = problem.solve(s, x, fx, f, tol=s.tol)
    dt = time.perf_counter() - t0
    return s.n_dof * sum(out["iters"]) / dt, dt, out["iters"], s


def host_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([1] + [p.get("num_threads", 1) for p in threadpool_info()])
    except Exception:
        return os.cpu_count() or 1


SWEEP_CONFIG = "c3_square_2048"
# bench_kernels entries -> the kernel they launch
KERNEL_NAMES = {"apply": "k_apply_tma<0>", "sgs_pre_update": "k_sgs_warp<ZERO,UPD> (pre-smoothing + r update)",
                "sgs_sweep": "k_sgs_warp<RZ> (post-smoothing sweep)", "residual": "k_apply_tma<1>",
                "p_update": "k_pcg_p (u, p update)"}
# FP64 work of the sweeps (FP64 instructions per step of the SASS loop,
# 2 flops per DFMA, per node swept, without the halo redundancy) and the FP64 peak measured
# with scripts/dfma_probe.cu on this pool's B200 (63.7 of 64 DFMA/clk/SM at 1965 MHz).
FP64_FLOP_PER_NODE = {"sgs_sweep": 315.0, "sgs_pre_update": 233.0}
FP64_PEAK_TFLOPS = 36.7


def inf_nodes(m, spec, nranks):
    """Nodes the timed kernels sweep on this rank (a strip: its share)."""
    return (spec.nelx + 1) * (spec.nely + 1) / nranks


def contrast_sweep(dev):
    """BASELINE configs[3]: the contrast-independence sweep.  For each
    E_min, one warm-up and one timed design pass (filter/project, basis, K_c assembly, PCG)
    on a fresh context; reports PCG iterations, PCG-only and whole-pass DOF*iter/s.  Runs
    after the timed region on rank 0 of a one-GPU run."""
    import torch
    from paper_1411_3923_b200 import Msfem
    base = W.CONFIGS[SWEEP_CONFIG]
    out = {"workload": SWEEP_CONFIG, "n_dof": base.n_dof, "rows": []}
    for emin in (1e-3, 1e-6, 1e-9):
        spec = base.replace(Emin=emin)
        m = Msfem.from_spec(spec, device=dev)
        x = torch.as_tensor(W.design_tile(spec), device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        for rep in range(2):
            ev[0].record(m.stream)
            m.filter_project(x)
            m.build_coarse_basis()
            m.assemble_coarse()
            ev[1].record(m.stream)
            its, comps, nc = m.pcg_solve(tol=spec.tol, max_it=20000)
            ev[2].record(m.stream)
            torch.cuda.synchronize(dev)
        setup_ms, pcg_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        out["rows"].append({"Emin": emin, "pcg_iters": its, "converged": not nc,
                            "pcg_ms": pcg_ms, "basis_assembly_ms": setup_ms,
                            "dof_iter_per_s_pcg": spec.n_dof * sum(its) / (pcg_ms / 1e3),
                            "dof_iter_per_s_pass": spec.n_dof * sum(its) / ((pcg_ms + setup_ms) / 1e3)})
        m.close()
        del m
        torch.cuda.empty_cache()
    its = [sum(r["pcg_iters"]) for r in out["rows"]]
    out["iters_spread_1e-6_to_1e-9"] = abs(its[2] - its[1]) / max(its[1:])
    return out


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


REF_CELLS = (4, 2)


def run_reference(args, spec):
    ws, rank, local = dist_setup()
    if rank != 0:
        return
    samples = []
    for i in range(args.warmup + args.steps):
        v, dt, its, s = oracle_sample(spec, REF_CELLS)
        if i >= args.warmup:
            samples.append((v, dt))
    value = float(np.mean([v for v, _ in samples]))
    ms = float(np.mean([dt for _, dt in samples])) * 1e3
    cores = host_threads()
    sample = (f"oracle (numpy/scipy fp64) full robust solve of the {spec.name} recipe on a "
              f"{s.nelx}x{s.nely} sub-grid ({s.n_dof} DOF, 3 realisations, iters {its})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": spec.name, "sample": cpu_sample_spec(spec, REF_CELLS).name},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, spec):
    import torch
    import torch.distributed as dist

    import paper_1411_3923_b200 as pkg
    from paper_1411_3923_b200 import Msfem

    ws, rank, local = dist_setup()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    # auto: strips when N > 1; "strips" forces the NCCL strip path even at N = 1 (a 1-rank
    # communicator: exercises the multi-GPU code path on one GPU)
    strips = (ws > 1 and args.mode == "auto") or args.mode == "strips"
    if strips:
        uid = [pkg.nccl_unique_id() if rank == 0 else None]
        if ws > 1:
            dist.broadcast_object_list(uid, src=0)
        m = Msfem(pkg.problem_from_spec(spec), W.fixed_mask(spec), W.load_vector(spec), device=dev,
                  rank=rank, nranks=ws, transport=pkg.MSF_TRANSPORT_NCCL, handle=uid[0])
    else:
        m = Msfem.from_spec(spec, device=dev)
    stream = m.stream
    x0 = W.design_tile(spec)
    xd = torch.as_tensor(x0, device=dev)
    xn = torch.empty_like(xd)
    tol, max_it = spec.tol, 5000

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        m.design_iteration(xd, xn, tol=tol, max_it=max_it)
    barrier()
    sampler = ClockSampler(local)
    sampler.start()
    m.launch_count(reset=True)
    iters_total = 0
    iters_step = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        its, comps, F, g = m.design_iteration(xd, xn, tol=tol, max_it=max_it)
        iters_total += sum(its)
        iters_step = its
    e1.record(stream)
    barrier()
    launches = m.launch_count()
    clocks = sampler.stop()
    t_ms = e0.elapsed_time(e1)
    t_max = t_ms
    if ws > 1:
        tt = torch.tensor([t_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        it_t = torch.tensor([iters_total], device=dev, dtype=torch.float64)
        dist.all_reduce(it_t, op=dist.ReduceOp.MAX if strips else dist.ReduceOp.SUM)
        iters_all = float(it_t.item())   # strips: one global solve (identical counts)
    else:
        iters_all = float(iters_total)
    value = spec.n_dof * iters_all / (t_max / 1e3)

    # ---- end to end through the C ABI with host (pinned) buffers
    xh = torch.as_tensor(x0).pin_memory()
    xnh = torch.empty_like(xh).pin_memory()
    m.design_iteration_host(xh, xnh, tol=tol, max_it=max_it)
    barrier()
    e2e_iters = 0
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        its, comps, F, g = m.design_iteration_host(xh, xnh, tol=tol, max_it=max_it)
        e2e_iters += sum(its)
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if ws > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
        it_t = torch.tensor([e2e_iters], device=dev, dtype=torch.float64)
        dist.all_reduce(it_t, op=dist.ReduceOp.MAX if strips else dist.ReduceOp.SUM)
        e2e_iters = float(it_t.item())
    e2e_value = spec.n_dof * e2e_iters / (e2e_ms / 1e3)
    nt = spec.tile_x * spec.tile_y
    h2d = nt * 8
    d2h = nt * 8 + spec.n_rhs * (4 + 8) + 16

    # ---- roofline of the dominant kernel (live CUDA-event timing, PCG launch config;
    # on a strip the kernels run on that rank's strip): all realisations active, and the
    # one-realisation configuration most PCG iterations of a step run in
    kb = m.bench_kernels(reps=20)
    os.environ["MSF_BENCH_NR"] = "1"
    kb1 = m.bench_kernels(reps=20)
    os.environ.pop("MSF_BENCH_NR", None)
    # kernels of one PCG iteration (msf_capi.cu enqueue_iteration): the largest time share
    per_iter_count = {"apply": 1, "sgs_pre_update": 1, "residual": 1, "restrict": 1,
                      "coarse_solve": 1, "prolong": 1, "sgs_sweep": 1, "p_update": 1}
    share = {k: kb[k][0] * n for k, n in per_iter_count.items()}
    dom = max(share, key=share.get)
    dom_ms, dom_bytes = kb[dom]
    peak, peak_src = hbm_peak()
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic = fp64_frac = None
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            traffic = tj.get(dom)
            fp64_frac = tj.get(dom + "_fp64_pipe_frac")
        except Exception:
            traffic = None
    fp64_roof = None
    if dom in FP64_FLOP_PER_NODE:
        nn_loc = inf_nodes(m, spec, ws if strips else 1)
        fl = FP64_FLOP_PER_NODE[dom] * nn_loc * spec.n_rhs
        fp64_roof = {"flop_per_launch": fl, "achieved_tflops": fl / (dom_ms / 1e3) / 1e12,
                     "peak_tflops": FP64_PEAK_TFLOPS,
                     "frac": fl / (dom_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                     "peak_source": "measured (scripts/dfma_probe.cu, dependent-free DFMA stream)"}
    inf = m.info()
    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        v, dt, its_c, s = oracle_sample(spec)
        cpu = {"value": v, "unit": UNIT, "cores": host_threads(), "kind": "oracle",
               "sample": f"oracle full robust solve (basis + 3 PCG) of the {spec.name} recipe on a "
                         f"{s.nelx}x{s.nely} sub-grid ({s.n_dof} DOF), iters {its_c}, {dt:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if strips and ws > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": spec.name, "n_dof": spec.n_dof, "grid": f"{spec.nelx}x{spec.nely}",
                   "realisations": spec.n_rhs, "coarse_cell": f"{spec.cx}x{spec.cy}",
                   "n_modes": spec.n_modes, "tile": f"{spec.tile_x}x{spec.tile_y}",
                   "tol": tol,
                   "parallelism": (f"{ws} strips (NCCL halos + all-reduces, distributed K_c chains + replicated interface system)"
                                   if strips else "single GPU" if ws == 1
                                   else f"{ws} independent replicas"),
                   "pcg_iters_per_step": iters_step, "n_agg_classes": inf["n_classes"],
                   "l2": f"inputs larger than L2: workspace {inf['workspace_bytes'] / 2**20:.0f} MiB > 126 MB"},
        "roofline": {"kernel": KERNEL_NAMES.get(dom, dom),
                     "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     # the sweeps are FP64-issue/latency-bound, not HBM-bound: ncu FP64 pipe share
                     "ncu_fp64_pipe_frac": fp64_frac,
                     "alg_bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms,
                     "peak_source": peak_src,
                     # the same launch against the FP64 roofline (the sweeps issue ~1 DFMA per 2
                     # instructions; ncu: FP64 pipe 45-57% busy incl. the halo redundancy)
                     "fp64": fp64_roof},
        # every timed kernel (all realisations active, PCG launch configuration): average ms per
        # launch-set, algorithmic GB/s and its fraction of the measured HBM peak
        "kernels": {k: {"ms": v[0],
                        "alg_GBps": v[1] / (v[0] / 1e3) / 1e9 if v[0] > 0 and v[1] > 0 else None,
                        "hbm_frac": v[1] / (v[0] / 1e3) / 1e9 / peak if v[0] > 0 and v[1] > 0 else None}
                    for k, v in kb.items()},
        "kernels_1rhs": {k: {"ms": v[0],
                             "hbm_frac": v[1] / (v[0] / 1e3) / 1e9 / peak if v[0] > 0 and v[1] > 0 else None}
                         for k, v in kb1.items()},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if ws == 1 and not args.no_sweep:
        m.close()
        del m
        torch.cuda.empty_cache()
        line["contrast_sweep"] = contrast_sweep(dev)
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the configs[3] contrast sweep after the timed region")
    ap.add_argument("--mode", default="auto", choices=["auto", "strips", "replicas"],
                    help="auto: strip partition when N > 1; strips: NCCL strip path even at N = 1; "
                         "replicas: independent copies per rank")
    args = ap.parse_args()
    spec = W.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, spec)
    else:
        run_ours(args, spec)


if __name__ == "__main__":
    main()
