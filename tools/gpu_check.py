"""Quick GPU parity + timing check (developer tool; uses the oracle as checker)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1604_02334_b200 import workloads as W, musr, objective, _lib
from oracle import musr_oracle as O

def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)

print("devices", _lib.device_count(), "fp64 peak TFLOP/s", _lib.fp64_peak_tflops(0), flush=True)
for name, kw in [("C1", {}), ("C2", dict(nbins=1 << 18)), ("C3", dict(n_hist=4, nbins=1 << 17))]:
    w = W.WORKLOADS[name](**kw)
    ds = W.synthesize(w)
    for kind, gf, of in [("chi2", musr.chi2, O.chi2), ("mlh", musr.mlh, O.mlh)]:
        t0 = time.perf_counter(); g = gf(ds, w.expr, w.params); t1 = time.perf_counter()
        g2 = gf(ds, w.expr, w.params); t2 = time.perf_counter()
        per = []
        o = of(ds, w.expr, w.params, per_dataset=per); t3 = time.perf_counter()
        sess = objective.session_for(ds, w.expr, musr.TAU_MU_US, len(w.params), objective.DeviceBackend())
        gp = sess.per_dataset()
        print(f"{name} {kind}: gpu={g!r} oracle={o!r} rel={rel(g, o):.3e} maxrel_per={max(rel(a,b) for a,b in zip(gp, per)):.3e} "
              f"repeat_equal={g == g2} first_call={1e3*(t1-t0):.1f}ms call={1e6*(t2-t1):.1f}us oracle={1e3*(t3-t2):.1f}ms", flush=True)

w = W.c2()
ds = W.synthesize(w)
sess = objective.session_for(ds, w.expr, musr.TAU_MU_US, len(w.params), objective.DeviceBackend())
v = musr.chi2(ds, w.expr, w.params)
for kind in (0, 1):
    ms = sess.time_evals(kind, 200, 0)
    kms = sess.time_evals(kind, 50, 1, True)
    nb = 8 * (1 << 20)
    print(f"C2 kind={kind}: graph {1e3*ms/200:.1f} us/eval  kernel(flushed) {1e3*kms/50:.1f} us  -> {nb/(ms/200*1e-3)/1e9:.1f} Gbins/s pipelined, "
          f"{nb*24/(kms/50*1e-3)/1e9:.0f} GB/s streamed(kernel)", flush=True)
t = time.perf_counter()
for _ in range(200): musr.chi2(ds, w.expr, w.params)
print(f"C2 sync drop-in: {1e6*(time.perf_counter()-t)/200:.1f} us/eval")
