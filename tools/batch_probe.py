"""Batched vs one-by-one evaluation throughput (developer tool, host-timed)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import workloads as W

for name in (sys.argv[1:] or ["C2"]):
    w = W.WORKLOADS[name]()
    ds = W.synthesize(w)
    nb = sum(len(d.counts) for d in ds)
    rng = np.random.default_rng(0)
    for kind, one, many in (("chi2", pkg.chi2, pkg.chi2_batch), ("mlh", pkg.mlh, pkg.mlh_batch)):
        for K in (1, 4, 8, 16):
            P = w.params * (1.0 + 0.01 * rng.standard_normal((K, len(w.params))))
            many(ds, w.expr, P)
            one(ds, w.expr, P[0])
            reps = max(3, 200 // K)
            t0 = time.perf_counter()
            for _ in range(reps):
                many(ds, w.expr, P)
            tb = (time.perf_counter() - t0) / reps
            t0 = time.perf_counter()
            for _ in range(reps):
                for p in P:
                    one(ds, w.expr, p)
            ts = (time.perf_counter() - t0) / reps
            print(f"{name} {kind} K={K:2d}: batch {1e6*tb/K:7.1f} us/point ({nb*K/tb/1e9:6.1f} Gbins/s)"
                  f"  single {1e6*ts/K:7.1f} us/point ({nb*K/ts/1e9:6.1f} Gbins/s)  x{ts/tb:.2f}", flush=True)
