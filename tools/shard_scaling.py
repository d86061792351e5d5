"""Single-GPU emulation of C4's strong scaling (developer tool): the objective
kernel on the shard one rank owns at N = 1, 2, 4, 8 GPUs (64/N datasets x 2^22
bins), device-timed with an L2 flush before every launch.  It bounds the
per-rank compute; the per-evaluation ncclAllReduce (1 KiB) is not included --
one GPU per call in this environment."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import workloads as W, objective

out = {}
for n_gpu in (1, 2, 4, 8):
    w = W.c4(n_hist=64 // n_gpu)
    dss = W.synthesize(w)
    pkg.chi2(dss, w.expr, w.params)
    sess = objective.session_for(dss, w.expr, pkg.TAU_MU_US, len(w.params), pkg.DeviceBackend())
    sess.time_evals(0, 5, 1, True)
    ms = sess.time_evals(0, 30, 1, True) / 30
    bins = sum(len(d.counts) for d in dss)
    out[n_gpu] = {"datasets_per_rank": len(dss), "bins_per_rank": bins, "kernel_us": 1e3 * ms,
                  "gbins_per_s_per_rank": bins / ms / 1e6}
    objective.clear_cache()
    del dss
t1 = out[1]["kernel_us"]
for n, r in out.items():
    r["implied_strong_scaling_efficiency"] = t1 / (n * r["kernel_us"])
print(json.dumps(out, indent=1))
