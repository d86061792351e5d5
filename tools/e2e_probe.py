"""Per-call latency of the drop-in objective (developer tool)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import workloads as W, objective

for name in ("C1", "C2"):
    w = W.WORKLOADS[name]()
    ds = W.synthesize(w)
    p = w.params.copy()
    pkg.chi2(ds, w.expr, p)
    sess = objective.session_for(ds, w.expr, pkg.TAU_MU_US, len(p), pkg.DeviceBackend())
    dev_ms = sess.time_evals(0, 200, 0)
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        pkg.chi2(ds, w.expr, p)
    t1 = time.perf_counter()
    for _ in range(n):
        sess.run(0, p)
    t2 = time.perf_counter()
    for _ in range(200):
        objective.session_for(ds, w.expr, pkg.TAU_MU_US, len(p), pkg.DeviceBackend())
    t3 = time.perf_counter()
    print(f"{name}: drop-in {1e6*(t1-t0)/n:.1f} us/call, session.run {1e6*(t2-t1)/n:.1f} us, "
          f"session lookup {1e6*(t3-t2)/200:.1f} us, device back-to-back {1e3*dev_ms/200:.1f} us")
