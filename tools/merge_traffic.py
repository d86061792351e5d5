"""Fold one measurement session's ncu summaries (tools/ncu_summary.py output,
keys like r2f_C4_chi2) into profiles/roofline_traffic.json (keys C4/chi2),
which bench.py reads for the physical-DRAM and executed-FP64 roofline lines.

    python tools/merge_traffic.py gpurun_out/r2f_roofline_traffic.json r2f
"""
import json, re, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
src, tag = Path(sys.argv[1]), sys.argv[2]
new = json.loads(src.read_text())
dst = ROOT / "profiles" / "roofline_traffic.json"
cur = json.loads(dst.read_text()) if dst.exists() else {}
for k, v in new.items():
    m = re.match(rf"{tag}_(\w+?)_(chi2|mlh)$", k)
    if not m:
        continue
    v["source"] = f"profiles/{tag}_ncu_{m.group(1)}_{m.group(2)}.txt"
    cur[f"{m.group(1)}/{m.group(2)}"] = v
dst.write_text(json.dumps(cur, indent=1) + "\n")
print(sorted(cur))
