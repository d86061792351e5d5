"""Per-region stall breakdown of an ncu --set full capture (developer tool).

    python tools/ncu_hotspots.py REPORT.ncu-rep [top_n]

Exports the SASS source page, prints total samples per stall reason, and the
top instructions by samples with their dominant stall reasons.
"""
import csv, io, subprocess, sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[col["# Samples"]])
    except ValueError:
        continue
    data.append((n, r[col["Address"]], r[col["Source"]].strip(), {s: int(r[col[s]] or 0) for s in stalls},
                 int(r[col["Instructions Executed"]] or 0)))
tot = Counter()
for n, a, src, st, ex in data:
    tot.update(st)
alls = sum(d[0] for d in data)
print(f"samples {alls}")
for k, v in tot.most_common():
    print(f"  {k:22s} {v:8d} {100 * v / max(alls, 1):5.1f}%")
print("top instructions:")
for i, (n, a, src, st, ex) in enumerate(sorted(data, key=lambda d: -d[0])[:top]):
    idx = [d[1] for d in data].index(a)
    dom = ", ".join(f"{k[6:]}={v}" for k, v in Counter(st).most_common(3) if v)
    print(f"  #{idx:5d} {n:6d} {src[:60]:60s} {dom}")
