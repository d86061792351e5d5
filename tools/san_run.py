"""Small multi-tile workload for compute-sanitizer runs (developer tool): one
C1-shaped dataset of 2^21 bins -> 512 tiles over the grid, so every CTA reuses
its pipeline stages (producer refills, look-ahead grabs, stage 2)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_02334_b200 import workloads as W, musr

w = W.c1(nbins=1 << 21)
ds = W.synthesize(w)
for kind in (musr.chi2, musr.mlh):
    print(kind.__name__, kind(ds, w.expr, w.params))
