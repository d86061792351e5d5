"""Small multi-tile workloads for compute-sanitizer runs (developer tool).

    python tools/san_run.py [c1|c2|small]

c1: one C1-shaped dataset of 2^21 bins -> 512 tiles over the grid, so every CTA
reuses its pipeline stages (producer refills, look-ahead grabs, stage 2 at exit).
c2: 8 C2-shaped datasets of 2^18 bins (512 tiles): datasets complete mid-launch,
so chi2 defers their stage 2 to CTAs out of tiles (claims by CAS).
small: one C1 dataset of 2^16 and one of 2^18 bins -- the small-problem tile
shapes (4 x 8 and 4 x 16 consumer warps, objective.small_problem_tile_shape)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_02334_b200 import workloads as W, musr

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
if case == "small":
    work = [W.c1(nbins=1 << 16), W.c1(nbins=1 << 18)]
else:
    work = [W.c1(nbins=1 << 21) if case == "c1" else W.c2(n_hist=8, nbins=1 << 18)]
for w in work:
    ds = W.synthesize(w)
    for kind in (musr.chi2, musr.mlh):
        print(kind.__name__, len(ds[0].counts), kind(ds, w.expr, w.params))
