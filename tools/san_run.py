"""Small multi-tile workloads for compute-sanitizer runs (developer tool).

    python tools/san_run.py [c1|c2]

c1: one C1-shaped dataset of 2^21 bins -> 512 tiles over the grid, so every CTA
reuses its pipeline stages (producer refills, look-ahead grabs, stage 2 at exit).
c2: 8 C2-shaped datasets of 2^18 bins (512 tiles): datasets complete mid-launch,
so chi2 defers their stage 2 to CTAs out of tiles (claims by CAS)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_02334_b200 import workloads as W, musr

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = W.c1(nbins=1 << 21) if case == "c1" else W.c2(n_hist=8, nbins=1 << 18)
ds = W.synthesize(w)
for kind in (musr.chi2, musr.mlh):
    print(kind.__name__, kind(ds, w.expr, w.params))
