"""Kernel-variant sweep (developer tool): NVRTC -D options x workloads."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1604_02334_b200 import workloads as W, musr, objective
from oracle import musr_oracle as O

variants = sys.argv[1].split(";") if len(sys.argv) > 1 else [""]
names = sys.argv[2].split(",") if len(sys.argv) > 2 else ["C2"]
data = {}
for n in names:  # "C1@262144": the workload at another bin count
    base, _, nb = n.partition("@")
    w = W.WORKLOADS[base](nbins=int(nb)) if nb else W.WORKLOADS[base]()
    data[n] = (w, W.synthesize(w))
ref = {}
for v in variants:
    cfg, _, opts = v.partition(":")
    pt, st, mb, cw = (cfg.split(",") + ["", "", "", ""])[:4]
    for key, val in (("MUSR_PT", pt), ("MUSR_STAGES", st), ("MUSR_MIN_BLOCKS", mb), ("MUSR_CWARPS", cw)):
        if val:
            os.environ[key] = val
        else:
            os.environ.pop(key, None)
    os.environ["MUSR_NVRTC_OPTS"] = opts
    objective.clear_cache()
    for n, (w, ds) in data.items():
        nb = sum(len(d.counts) for d in ds)
        s = objective.session_for(ds, w.expr, musr.TAU_MU_US, len(w.params), objective.DeviceBackend())
        out = []
        for kind, f in ((0, musr.chi2), (1, musr.mlh)):
            val = f(ds, w.expr, w.params)
            key = (n, kind)
            if key not in ref:
                ref[key] = val
            fl = int(os.environ.get("MUSR_FLUSH", "1"))
            s.time_evals(kind, 20, 1, fl)
            ms_k = s.time_evals(kind, 100, 1, fl) / 100
            ms_g = s.time_evals(kind, 400, 0) / 400
            out.append(f"{'chi2' if kind == 0 else 'mlh'} kernel {1e3*ms_k:7.1f}us ({nb/ms_k/1e6:6.1f} Gbins/s) graph {1e3*ms_g:7.1f}us ({nb/ms_g/1e6:6.1f}) same={val == ref[key]}")
        print(f"[{v or 'default'}] {n} tiles={s.n_tiles()} | " + " | ".join(out), flush=True)
