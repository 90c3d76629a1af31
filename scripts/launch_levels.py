"""Prints the last N launches (name, grid, device ns) of an ncu --csv launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
tot = 0.0
for d in data[-n:]:
    nm = d["Kernel Name"].split("(")[0].split("::")[-1]
    tot += float(d["Metric Value"])
    print(f"{nm:40s} {d.get('Grid Size', ''):>16s} {float(d['Metric Value']) / 1e3:8.1f} us")
print(f"total {tot / 1e3:.1f} us over {min(n, len(data))} launches")
