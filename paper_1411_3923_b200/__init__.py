"""B200-native hot path of arxiv 1411.3923 (spectral-MsFEM preconditioned PCG for robust
microstructural topology optimisation).

This package is a thin binding over the C-ABI library ``libmsfem_b200.so``
(``include/msfem_b200.h``): argument marshalling only -- every step of the path runs in the
library's CUDA kernels.  PyTorch provides device memory (the workspace and vectors) and the
CUDA stream.  There is no CPU fallback: importing ``Msfem`` without the built library or
without an sm_100 device raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSF_LIB_PATH", os.path.join(HERE, "libmsfem_b200.so"))

MSF_OK, MSF_ERR_ARG, MSF_ERR_CUDA, MSF_ERR_STATE, MSF_ERR_NOCONV, MSF_ERR_FACTOR, MSF_ERR_SPACE = \
    0, -1, -2, -3, -4, -5, -6
MSF_TRANSPORT_NCCL, MSF_TRANSPORT_GROUP = 1, 2
MAX_RHS = 4

# every symbol declared in include/msfem_b200.h (checked by tests/test_abi.py)
EXPORTS = [
    "msf_workspace_bytes", "msf_setup_mesh", "msf_destroy", "msf_set_stream", "msf_last_error",
    "msf_filter_project", "msf_set_physical", "msf_build_coarse_basis", "msf_assemble_coarse",
    "msf_pcg_solve", "msf_sensitivities", "msf_oc_update", "msf_design_iteration",
    "msf_design_iteration_host", "msf_matvec", "msf_precond_apply", "msf_sgs", "msf_sgs_ex",
    "msf_coarse_solve", "msf_get_basis", "msf_get_coarse_blocks", "msf_get_physical",
    "msf_info", "msf_launch_count", "msf_bench_kernels",
    "msf_strip_bounds", "msf_dist_workspace_bytes", "msf_dist_setup", "msf_nccl_unique_id",
    "msf_group_create", "msf_group_destroy", "msf_group_assemble_coarse", "msf_group_coarse_solve", "msf_group_precond_apply", "msf_group_pcg_solve", "msf_group_sensitivities",
    "msf_get_solution",
]


class MsfProblem(ctypes.Structure):
    _fields_ = [("nelx", ctypes.c_int32), ("nely", ctypes.c_int32),
                ("cx", ctypes.c_int32), ("cy", ctypes.c_int32),
                ("n_modes", ctypes.c_int32), ("tile_x", ctypes.c_int32),
                ("tile_y", ctypes.c_int32), ("n_rhs", ctypes.c_int32),
                ("dilated", ctypes.c_int32), ("eig_max_iter", ctypes.c_int32),
                ("nu", ctypes.c_double), ("E0", ctypes.c_double), ("Emin", ctypes.c_double),
                ("penal", ctypes.c_double), ("rmin", ctypes.c_double), ("beta", ctypes.c_double),
                ("eta", ctypes.c_double * MAX_RHS), ("lam_threshold", ctypes.c_double),
                ("eig_tol", ctypes.c_double)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Loads the C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_1411_3923_b200.build` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    P, I, D, V = ctypes.POINTER, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    i32p, dp, i64p = P(ctypes.c_int32), P(ctypes.c_double), P(ctypes.c_int64)
    sig = {
        "msf_workspace_bytes": [P(MsfProblem), V, P(ctypes.c_size_t)],
        "msf_setup_mesh": [P(MsfProblem), V, V, V, ctypes.c_size_t, V, P(V)],
        "msf_destroy": [V], "msf_set_stream": [V, V],
        "msf_filter_project": [V, V], "msf_set_physical": [V, I, V],
        "msf_build_coarse_basis": [V], "msf_assemble_coarse": [V],
        "msf_pcg_solve": [V, I, D, I, V, i32p, dp],
        "msf_sensitivities": [V, D, D, V, V, dp, dp, dp],
        "msf_oc_update": [V, V, V, V, D, D, V],
        "msf_design_iteration": [V, V, V, D, I, D, D, D, i32p, dp, dp, dp],
        "msf_design_iteration_host": [V, V, V, D, I, D, D, D, i32p, dp, dp, dp],
        "msf_matvec": [V, I, V, V], "msf_precond_apply": [V, I, V, V], "msf_sgs": [V, I, V, V],
        "msf_sgs_ex": [V, I, V, V, I],
        "msf_coarse_solve": [V, I, V, V], "msf_get_basis": [V, V, V, V],
        "msf_get_coarse_blocks": [V, I, V, V], "msf_get_physical": [V, I, V, V],
        "msf_info": [V, i64p], "msf_launch_count": [V, i64p, I],
        "msf_bench_kernels": [V, I, dp, dp],
        "msf_strip_bounds": [P(MsfProblem), I, I, i32p],
        "msf_dist_workspace_bytes": [P(MsfProblem), V, I, I, P(ctypes.c_size_t)],
        "msf_dist_setup": [P(MsfProblem), V, V, I, I, I, V, V, ctypes.c_size_t, V, P(V)],
        "msf_nccl_unique_id": [V], "msf_get_solution": [V, I, V],
        "msf_group_create": [I, P(V)], "msf_group_destroy": [V],
        "msf_group_assemble_coarse": [V],
        "msf_group_coarse_solve": [V, I, V, V],
        "msf_group_precond_apply": [V, I, V, V],
        "msf_group_pcg_solve": [V, I, D, I, i32p, dp],
        "msf_group_sensitivities": [V, D, D, V, V, dp, dp, dp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.msf_last_error.argtypes = [V]
    lib.msf_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


class MsfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"msf error {code}: {msg}")
        self.code = code


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def problem_from_spec(spec) -> MsfProblem:
    """Marshals a workloads.ProblemSpec into the C struct."""
    p = MsfProblem()
    p.nelx, p.nely, p.cx, p.cy = spec.nelx, spec.nely, spec.cx, spec.cy
    p.n_modes, p.tile_x, p.tile_y = spec.n_modes, spec.tile_x, spec.tile_y
    p.n_rhs, p.dilated, p.eig_max_iter = len(spec.etas), spec.dilated, 0
    p.nu, p.E0, p.Emin, p.penal = spec.nu, spec.E0, spec.Emin, spec.penal
    p.rmin, p.beta = spec.rmin, spec.beta
    for k, e in enumerate(spec.etas):
        p.eta[k] = e
    p.lam_threshold = spec.lam_threshold if np.isfinite(spec.lam_threshold) else 0.0
    p.eig_tol = 0.0
    return p


def strip_bounds(problem: MsfProblem, rank: int, nranks: int) -> dict:
    """Strip of `rank` (msf_strip_bounds; host only, no GPU needed)."""
    lib = load_library()
    b = (ctypes.c_int32 * 8)()
    rc = lib.msf_strip_bounds(ctypes.byref(problem), rank, nranks, b)
    if rc != MSF_OK:
        raise MsfError(rc, lib.msf_last_error(None).decode())
    keys = ["own0", "own1", "gox", "ncols", "e0", "e1", "C0", "C1"]
    return dict(zip(keys, list(b)))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the caller broadcasts it)."""
    lib = load_library()
    buf = (ctypes.c_uint8 * 128)()
    rc = lib.msf_nccl_unique_id(buf)
    if rc != MSF_OK:
        raise MsfError(rc, lib.msf_last_error(None).decode())
    return bytes(buf)


class Msfem:
    """One problem instance on the current CUDA device (C-ABI context + torch workspace).

    rank/nranks/transport/handle: strip partition (msf_dist_setup); transport
    MSF_TRANSPORT_NCCL takes the 128-byte unique id as handle, MSF_TRANSPORT_GROUP an
    MsfemGroup (use MsfemGroup.create instead of calling this directly)."""

    def __init__(self, problem: MsfProblem, fixed_mask: np.ndarray, load: np.ndarray,
                 device=None, stream=None, rank=0, nranks=1, transport=0, handle=None):
        import torch
        self.torch = torch
        self.lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.problem = problem
        self.fixed = np.ascontiguousarray(fixed_mask, dtype=np.uint8)
        self.load = np.ascontiguousarray(load, dtype=np.float64)
        self.rank, self.nranks, self.transport = rank, nranks, transport
        nbytes = ctypes.c_size_t()
        fx = self.fixed.ctypes.data_as(ctypes.c_void_p)
        if transport:
            self._check(self.lib.msf_dist_workspace_bytes(ctypes.byref(problem), fx, rank, nranks,
                                                          ctypes.byref(nbytes)), None)
            self.bounds = strip_bounds(problem, rank, nranks)
        else:
            self._check(self.lib.msf_workspace_bytes(ctypes.byref(problem), fx,
                                                     ctypes.byref(nbytes)), None)
            self.bounds = {"own0": 0, "own1": problem.nelx + 1, "gox": 0,
                           "ncols": problem.nelx + 1, "e0": 0, "e1": problem.nelx,
                           "C0": 0, "C1": problem.nelx // problem.cx}
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = ctypes.c_void_p()
        ld = self.load.ctypes.data_as(ctypes.c_void_p)
        st = ctypes.c_void_p(self.stream.cuda_stream)
        if transport:
            if transport == MSF_TRANSPORT_NCCL:
                self._id_buf = (ctypes.c_uint8 * 128).from_buffer_copy(handle)
                h = ctypes.cast(self._id_buf, ctypes.c_void_p)
            else:
                h = handle
            self._check(self.lib.msf_dist_setup(ctypes.byref(problem), fx, ld, rank, nranks,
                                                transport, h, _ptr(self.workspace), nbytes.value,
                                                st, ctypes.byref(ctx)), None)
        else:
            self._check(self.lib.msf_setup_mesh(ctypes.byref(problem), fx, ld,
                                                _ptr(self.workspace), nbytes.value, st,
                                                ctypes.byref(ctx)), None)
        self.ctx = ctx
        self.n_dof_local = 2 * self.bounds["ncols"] * (problem.nely + 1)
        self.n_rhs = problem.n_rhs
        self.n_dof = 2 * (problem.nelx + 1) * (problem.nely + 1)
        self.n_el = problem.nelx * problem.nely
        self.n_tile = problem.tile_x * problem.tile_y

    @classmethod
    def from_spec(cls, spec, **kw):
        import workloads as W
        return cls(problem_from_spec(spec), W.fixed_mask(spec), W.load_vector(spec), **kw)

    def _check(self, rc, ctx="self", allow_noconv=False):
        if rc == MSF_OK or (allow_noconv and rc == MSF_ERR_NOCONV):
            return rc
        c = self.ctx if ctx == "self" else ctx
        msg = self.lib.msf_last_error(c)
        raise MsfError(rc, msg.decode() if msg else "")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.msf_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- boundary calls (§8(b))
    def filter_project(self, x_tile):
        self._check(self.lib.msf_filter_project(self.ctx, _ptr(x_tile)))

    def set_physical(self, rhs, xbar_el):
        self._check(self.lib.msf_set_physical(self.ctx, rhs, _ptr(xbar_el)))

    def build_coarse_basis(self):
        self._check(self.lib.msf_build_coarse_basis(self.ctx))

    def assemble_coarse(self):
        self._check(self.lib.msf_assemble_coarse(self.ctx))

    def pcg_solve(self, n_rhs=None, tol=1e-8, max_it=2000, u=None):
        n = self.n_rhs if n_rhs is None else n_rhs
        iters = (ctypes.c_int32 * n)()
        comp = (ctypes.c_double * n)()
        rc = self._check(self.lib.msf_pcg_solve(self.ctx, n, tol, max_it, _ptr(u), iters, comp),
                         allow_noconv=True)
        return list(iters), list(comp), rc == MSF_ERR_NOCONV

    def sensitivities(self, kappa=1.0, volfrac=0.5, dF=None, dg=None):
        F, g = ctypes.c_double(), ctypes.c_double()
        comp = (ctypes.c_double * self.n_rhs)()
        self._check(self.lib.msf_sensitivities(self.ctx, kappa, volfrac, _ptr(dF), _ptr(dg),
                                               ctypes.byref(F), ctypes.byref(g), comp))
        return F.value, g.value, list(comp)

    def oc_update(self, x, dF, dg, volfrac=0.5, move=0.2, x_new=None):
        self._check(self.lib.msf_oc_update(self.ctx, _ptr(x), _ptr(dF), _ptr(dg), volfrac, move,
                                           _ptr(x_new)))

    def design_iteration(self, x, x_new, tol=1e-8, max_it=2000, kappa=1.0, volfrac=0.5,
                         move=0.2):
        iters = (ctypes.c_int32 * self.n_rhs)()
        comp = (ctypes.c_double * self.n_rhs)()
        F, g = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.msf_design_iteration(self.ctx, _ptr(x), _ptr(x_new), tol, max_it,
                                                  kappa, volfrac, move, iters, comp,
                                                  ctypes.byref(F), ctypes.byref(g)),
                    allow_noconv=True)
        return list(iters), list(comp), F.value, g.value

    def design_iteration_host(self, x_host: np.ndarray, x_new_host: np.ndarray, tol=1e-8,
                              max_it=2000, kappa=1.0, volfrac=0.5, move=0.2):
        iters = (ctypes.c_int32 * self.n_rhs)()
        comp = (ctypes.c_double * self.n_rhs)()
        F, g = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.msf_design_iteration_host(
            self.ctx, ctypes.c_void_p(x_host.ctypes.data if isinstance(x_host, np.ndarray) else x_host.data_ptr()),
            ctypes.c_void_p(x_new_host.ctypes.data if isinstance(x_new_host, np.ndarray) else x_new_host.data_ptr()),
            tol, max_it, kappa, volfrac, move, iters, comp, ctypes.byref(F), ctypes.byref(g)),
            allow_noconv=True)
        return list(iters), list(comp), F.value, g.value

    # ------------------------------------------------------------- diagnostics
    def matvec(self, rhs, x, y):
        self._check(self.lib.msf_matvec(self.ctx, rhs, _ptr(x), _ptr(y)))

    def precond_apply(self, rhs, r, z):
        self._check(self.lib.msf_precond_apply(self.ctx, rhs, _ptr(r), _ptr(z)))

    def sgs(self, rhs, r, z, zero_start=False, phases=False):
        flags = (1 if zero_start else 0) | (2 if phases else 0)
        if flags:
            self._check(self.lib.msf_sgs_ex(self.ctx, rhs, _ptr(r), _ptr(z), flags))
        else:
            self._check(self.lib.msf_sgs(self.ctx, rhs, _ptr(r), _ptr(z)))

    def coarse_solve(self, rhs, b, c):
        self._check(self.lib.msf_coarse_solve(self.ctx, rhs, _ptr(b), _ptr(c)))

    def info(self):
        a = (ctypes.c_int64 * 16)()
        self._check(self.lib.msf_info(self.ctx, a))
        keys = ["n_dof", "n_el", "n_agg", "n_classes", "ncx", "ncy", "m", "coarse_slots",
                "box_nodes", "eig_iters", "it0", "it1", "it2", "it3", "pcg_iter_launches",
                "workspace_bytes"]
        return dict(zip(keys, list(a)))

    def get_basis(self):
        inf = self.info()
        p = self.problem
        per = p.n_modes * inf["box_nodes"] * 2
        phi = np.zeros(inf["n_agg"] * per)
        nk = np.zeros(inf["n_agg"], dtype=np.int32)
        lam = np.zeros(inf["n_agg"] * p.n_modes)
        self._check(self.lib.msf_get_basis(self.ctx, phi.ctypes.data_as(ctypes.c_void_p),
                                           nk.ctypes.data_as(ctypes.c_void_p),
                                           lam.ctypes.data_as(ctypes.c_void_p)))
        return (phi.reshape(inf["n_agg"], p.n_modes, 2 * p.cx + 1, 2 * p.cy + 1, 2), nk,
                lam.reshape(inf["n_agg"], p.n_modes))

    def get_coarse_blocks(self, rhs):
        inf = self.info()
        m, nb = inf["m"], inf["ncx"] + 1
        D = np.zeros((nb, m, m))
        U = np.zeros((nb, m, m))
        self._check(self.lib.msf_get_coarse_blocks(self.ctx, rhs, D.ctypes.data_as(ctypes.c_void_p),
                                                   U.ctypes.data_as(ctypes.c_void_p)))
        return D, U

    def get_solution(self, n_rhs=None):
        """u of the last PCG solve (device [n_rhs * n_dof_local]; the strip on a strip context)."""
        n = self.n_rhs if n_rhs is None else n_rhs
        u = self.torch.empty(n * self.n_dof_local, dtype=self.torch.float64, device=self.device)
        self._check(self.lib.msf_get_solution(self.ctx, n, _ptr(u)))
        return u

    def get_physical(self, rhs, E_el=None, xbar_tile=None):
        self._check(self.lib.msf_get_physical(self.ctx, rhs, _ptr(E_el), _ptr(xbar_tile)))

    def launch_count(self, reset=False):
        c = ctypes.c_int64()
        self._check(self.lib.msf_launch_count(self.ctx, ctypes.byref(c), 1 if reset else 0))
        return c.value

    def bench_kernels(self, reps=20):
        """Per-kernel average ms and algorithmic bytes per launch (see msf_bench_kernels)."""
        ms = (ctypes.c_double * 15)()
        by = (ctypes.c_double * 15)()
        self._check(self.lib.msf_bench_kernels(self.ctx, reps, ms, by))
        names = ["apply", "sgs_sweep", "restrict", "coarse_solve", "prolong", "residual",
                 "vcycle", "pcg_iteration", "sgs_pre_update", "p_update", "assemble_local",
                 "assemble_top", "coarse_fwd_local", "coarse_top", "coarse_back_local"]
        return {n: (ms[i], by[i]) for i, n in enumerate(names)}


class MsfemGroup:
    """All ranks of a strip partition as contexts of this process on one device
    (MSF_TRANSPORT_GROUP): replicated steps run per rank, the communicating steps
    (K_c assembly, PCG, sensitivities, the coarse-solve / V-cycle diagnostics) through the
    group entry points.  Proves the partitioned path on a
    single GPU; production multi-GPU runs use one process per GPU with NCCL."""

    def __init__(self, problem: MsfProblem, fixed_mask, load, nranks, stream=None):
        import torch
        self.lib = load_library()
        g = ctypes.c_void_p()
        rc = self.lib.msf_group_create(nranks, ctypes.byref(g))
        if rc != MSF_OK:
            raise MsfError(rc, self.lib.msf_last_error(None).decode())
        self.g = g
        self.problem = problem
        self.nranks = nranks
        st = stream if stream is not None else torch.cuda.current_stream()
        self.ranks = [Msfem(problem, fixed_mask, load, stream=st, rank=r, nranks=nranks,
                            transport=MSF_TRANSPORT_GROUP, handle=g) for r in range(nranks)]
        self.n_rhs = problem.n_rhs

    @classmethod
    def from_spec(cls, spec, nranks, **kw):
        import workloads as W
        return cls(problem_from_spec(spec), W.fixed_mask(spec), W.load_vector(spec), nranks, **kw)

    def _check(self, rc, allow_noconv=False):
        if rc == MSF_OK or (allow_noconv and rc == MSF_ERR_NOCONV):
            return rc
        raise MsfError(rc, self.lib.msf_last_error(None).decode())

    def filter_project(self, x_tile):
        for m in self.ranks:
            m.filter_project(x_tile)

    def set_physical(self, rhs, xbar_el):
        for m in self.ranks:
            m.set_physical(rhs, xbar_el)

    def build_coarse_basis(self):
        for m in self.ranks:
            m.build_coarse_basis()

    def assemble_coarse(self):
        self._check(self.lib.msf_group_assemble_coarse(self.g))

    def coarse_solve(self, rhs, b, x=None):
        """Distributed K_c^{-1} b (parity diagnostic); b, x: device [n_coarse_slots]."""
        import torch
        x = torch.empty_like(b) if x is None else x
        self._check(self.lib.msf_group_coarse_solve(self.g, rhs, _ptr(b), _ptr(x)))
        return x

    def precond_apply(self, rhs, r, z=None):
        """Partitioned V-cycle z = M^{-1} r (parity diagnostic); r, z: device [n_dof]."""
        import torch
        z = torch.zeros_like(r) if z is None else z
        self._check(self.lib.msf_group_precond_apply(self.g, rhs, _ptr(r), _ptr(z)))
        return z

    def pcg_solve(self, n_rhs=None, tol=1e-8, max_it=2000):
        n = self.n_rhs if n_rhs is None else n_rhs
        iters = (ctypes.c_int32 * n)()
        comp = (ctypes.c_double * n)()
        rc = self._check(self.lib.msf_group_pcg_solve(self.g, n, tol, max_it, iters, comp),
                         allow_noconv=True)
        return list(iters), list(comp), rc == MSF_ERR_NOCONV

    def sensitivities(self, kappa=1.0, volfrac=0.5, dF=None, dg=None):
        F, g = ctypes.c_double(), ctypes.c_double()
        comp = (ctypes.c_double * self.n_rhs)()
        self._check(self.lib.msf_group_sensitivities(self.g, kappa, volfrac, _ptr(dF), _ptr(dg),
                                                     ctypes.byref(F), ctypes.byref(g), comp))
        return F.value, g.value, list(comp)

    def gather_solution(self, n_rhs=None):
        """Global u [n_rhs, n_dof] (device) assembled from the ranks' owned node columns."""
        import torch
        n = self.n_rhs if n_rhs is None else n_rhs
        p = self.problem
        nny = p.nely + 1
        out = torch.zeros(n, (p.nelx + 1) * nny * 2, dtype=torch.float64, device="cuda")
        for m in self.ranks:
            b = m.bounds
            loc = m.get_solution(n).view(n, -1)
            lo = (b["own0"] - b["gox"]) * nny * 2
            hi = (b["own1"] - b["gox"]) * nny * 2
            out[:, b["own0"] * nny * 2:b["own1"] * nny * 2] = loc[:, lo:hi]
        return out

    def close(self):
        for m in self.ranks:
            m.close()
        if getattr(self, "g", None):
            self.lib.msf_group_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
