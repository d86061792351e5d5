"""Workload runner for ncu captures: build a session, run N kernel launches."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1604_02334_b200 import workloads as W, musr, objective

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C2")
ap.add_argument("--kind", type=int, default=0)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
w = W.WORKLOADS[a.workload]()
ds = W.synthesize(w)
s = objective.session_for(ds, w.expr, musr.TAU_MU_US, len(w.params), objective.DeviceBackend())
(musr.chi2 if a.kind == 0 else musr.mlh)(ds, w.expr, w.params)
print("ms", s.time_evals(a.kind, a.iters, 1, True) / a.iters)
