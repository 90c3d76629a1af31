"""Per-PCG-iteration kernel breakdown from an ncu launch list
(ncu --metrics gpu__time_duration.sum --csv --log-file X.csv ...): markdown table.
With --all: every launch of the list (e.g. one whole bench step), share of the total.
Reads .csv or .csv.gz."""
import collections
import csv
import gzip
import sys


def main(path, whole=False):
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    rows = list(csv.reader(f))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    seq = []
    for r in rows[hdr + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        u = r[ui]
        v = v * 1e3 if u in ("us", "usecond") else (v * 1e6 if u in ("ms", "msecond") else v)
        seq.append((r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", ""), v))
    if whole:
        agg, cnt = collections.defaultdict(float), collections.defaultdict(int)
        for k, v in seq:
            agg[k.split("<")[0]] += v
            cnt[k.split("<")[0]] += 1
        tot = sum(agg.values())
        print(f"{len(seq)} launches; serialised kernel time {tot / 1e6:.2f} ms\n")
        print("| kernel | ms | launches | share |")
        print("|---|---|---|---|")
        for k, v in sorted(agg.items(), key=lambda x: -x[1]):
            print(f"| {k} | {v / 1e6:.3f} | {cnt[k]} | {v / tot * 100:.1f}% |")
        return
    starts = [i for i, (k, _) in enumerate(seq)
              if k.startswith(("k_apply<0", "k_apply_direct<0", "k_apply_tma<0", "k_apply_sw<0"))]
    agg, cnt, tot = collections.defaultdict(float), collections.defaultdict(int), 0.0
    for a, b in zip(starts[:-1], starts[1:]):
        for k, v in seq[a:b]:
            kk = k.split("<")[0]
            agg[kk] += v
            cnt[kk] += 1
            tot += v
    n = len(starts) - 1
    print(f"{n} PCG iterations; kernel time per iteration (serialised under ncu): {tot / n / 1e3:.1f} us\n")
    print("| kernel | us / iteration | launches / iteration | share |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"| {k} | {v / n / 1e3:.1f} | {cnt[k] / n:.0f} | {v / tot * 100:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], "--all" in sys.argv[2:])
