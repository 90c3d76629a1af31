"""bench.py keeps the driver's JSON-line contract: the reference arm (the oracle on the host,
CPU) and our arm (GPU) each print one line with the keys the driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "0", "--config", "c0_cantilever_96x48")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]


@pytest.mark.gpu
def test_our_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = run_bench("--steps", "2", "--warmup", "3", "--no-cpu-baseline", timeout=1200)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["config"]["workload"] == "c4_mbb_5120x2560" and d["config"]["n_dof"] == 26229762
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] <= 1.2
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e2e = d["e2e"]
    assert e2e["unit"] == d["unit"] and e2e["value"] > 0
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 1000
    its = d["config"]["pcg_iters_per_step"]
    assert len(its) == 3 and its[0] > its[1] > its[2] > 0   # eroded > intermediate > dilated
    for tab in (d["kernels"], d["kernels_1rhs"]):
        assert {"apply", "sgs_sweep", "sgs_pre_update", "vcycle", "pcg_iteration"} <= set(tab)
    sw = d["contrast_sweep"]
    assert sw["workload"] == "c3_square_2048" and [r["Emin"] for r in sw["rows"]] == [1e-3, 1e-6, 1e-9]
    assert all(r["converged"] and r["dof_iter_per_s_pcg"] > 0 for r in sw["rows"])
    # iteration counts nearly flat in the contrast
    assert sw["iters_spread_1e-6_to_1e-9"] <= 0.15


def test_reference_arm_under_torchrun_two_ranks():
    """The driver's N > 1 launch of the reference arm: rank 0 alone prints one line, every
    rank exits 0."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "0", "--config", "c0_cantilever_96x48"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_our_arm_strips_mode_one_rank():
    """The NCCL strip path (1-rank communicator) through bench.py: same workload, iteration
    counts and a valid line."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    args = ("--config", "c1_mbb_1024x512", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-sweep")
    d = run_bench("--mode", "strips", *args)
    s = run_bench(*args)
    assert all(abs(a - b) <= 1 for a, b in zip(d["config"]["pcg_iters_per_step"], s["config"]["pcg_iters_per_step"]))
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 1000
