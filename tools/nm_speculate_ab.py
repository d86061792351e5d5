"""A/B of the speculative Nelder-Mead batch (musr_nm.cpp nm_core `speculate`):
this package's minimize() on a workload with MUSR_NM_SPECULATE=0 / 1, wall time
per fit (best of 3, session built outside), evaluation count, and whether the
fitted parameters are bit-identical.

    python tools/nm_speculate_ab.py [workload[@nbins] ...]     # default C1 C1@262144 C2
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import workloads as W

names = sys.argv[1:] or ["C1", "C1@262144", "C2"]
for name in names:
    base, _, nb = name.partition("@")
    w = W.WORKLOADS[base](nbins=int(nb)) if nb else W.WORKLOADS[base]()
    dss = W.synthesize(w)
    n = len(w.params)
    fixed = np.zeros(n, dtype=bool)
    for j in range(len(dss)):                      # N0 / Nbkg fixed, as in the C5 fit
        fixed[dss[j].n0_slot] = fixed[dss[j].nbkg_slot] = True
    start = w.params * np.where(fixed, 1.0, 1.07)
    steps = np.maximum(np.abs(w.params) * 0.05, 1e-3)
    pkg.chi2(dss, w.expr, start)                   # session outside the timed region
    out = {"workload": name, "bins": int(sum(len(d.counts) for d in dss))}
    res = {}
    for spec in ("0", "1"):
        os.environ["MUSR_NM_SPECULATE"] = spec
        best = None
        for _ in range(3):
            ps = pkg.ParameterSet(values=start.copy(), names=[f"p{i}" for i in range(n)],
                                  step_sizes=steps.copy(), fixed=fixed.copy())
            t0 = time.perf_counter()
            r = pkg.minimize("chi2", dss, w.expr, ps)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        res[spec] = r
        out[f"fit_ms_spec{spec}"] = 1e3 * best
        out[f"evals_spec{spec}"] = r.objective_evaluations
        out[f"iterations_spec{spec}"] = r.iterations
    os.environ.pop("MUSR_NM_SPECULATE")
    out["bitwise_equal"] = bool(np.array_equal(res["0"].best_parameters.values,
                                               res["1"].best_parameters.values)
                                and res["0"].objective_value == res["1"].objective_value)
    print(json.dumps(out), flush=True)
