"""Summarise ncu --set full reports (raw page) into a markdown table row per kernel.
Columns: time, DRAM read / write, DRAM % of peak, warps active %, issue active %, FP64 pipe %,
DMMA (fp64 tensor) pipe %, L1 / L2 hit rates, registers, grid, top stall reasons."""
import csv, io, subprocess, sys
KEYS = [("gpu__time_duration.sum", "us", 1e-3), ("dram__bytes_read.sum", "MB", 1e-6),
        ("dram__bytes_write.sum", "MB", 1e-6),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "%", 1),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "%", 1),
        ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "%", 1),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "%", 1),
        ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "%", 1),
        ("l1tex__t_sector_hit_rate.pct", "%", 1), ("lts__t_sector_hit_rate.pct", "%", 1),
        ("launch__registers_per_thread", "", 1), ("launch__grid_size", "", 1)]
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "math_pipe_throttle",
          "lg_throttle", "mio_throttle", "not_selected", "selected"]
def units_scale(u, v):
    u = u.strip()
    if u in ("nsecond", "ns"): return v
    if u in ("usecond", "us"): return v * 1e3
    if u in ("msecond", "ms"): return v * 1e6
    if u in ("byte",): return v
    if u in ("Kbyte", "KB"): return v * 1e3
    if u in ("Mbyte", "MB"): return v * 1e6
    if u in ("Gbyte", "GB"): return v * 1e9
    return v
for path in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:60]
        cells = []
        for k, u, sc in KEYS:
            if k not in hdr:
                cells.append("-")
                continue
            i = hdr.index(k)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                cells.append("-")
                continue
            if u in ("us", "MB"):
                v = units_scale(units[i], v) * (1e-3 if u == "us" else 1e-6)
            cells.append(f"{v:.3g}")
        st = []
        tot = 0.0
        vals = {}
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in hdr:
                vals[s] = float(r[hdr.index(k)].replace(",", "") or 0)
                tot += vals[s]
        top = sorted(vals.items(), key=lambda kv: -kv[1])[:3]
        print(f"| {name} | " + " | ".join(cells) + " | " + ", ".join(f"{k} {v/tot*100:.0f}%" for k, v in top) + " |")
