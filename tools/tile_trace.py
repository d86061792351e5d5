"""Per-tile timeline of one objective launch (developer tool, MUSR_TRACE=1):
for the last tiles of the launch, when each was published (grabbed) and folded,
by which CTA -- the C2 tail analysis in DESIGN.md."""
import ctypes as C, os, sys
from pathlib import Path
os.environ["MUSR_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1604_02334_b200 import workloads as W, musr, objective, _lib

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
w = W.WORKLOADS[name]()
ds = W.synthesize(w)
s = objective.session_for(ds, w.expr, musr.TAU_MU_US, len(w.params), objective.DeviceBackend())
musr.chi2(ds, w.expr, w.params)
ms = s.time_evals(0, 3, 1, int(os.environ.get("MUSR_FLUSH", "1"))) / 3
nt = s.n_tiles()
sms = _lib.device_sms(0) if hasattr(_lib, "device_sms") else 148
cap = sms * 32 + 3 * nt
buf = (C.c_uint64 * cap)()
n = C.c_int()
_lib.check(s._lib.musr_debug_trace(s._handle, 0, buf, cap, C.byref(n)), s._handle, "trace")
a = np.array(buf, dtype=np.int64)
start = a[: 4 * n.value].reshape(-1, 4)[:, 0]
t0 = start[start > 0].min()
tt = a[sms * 32: sms * 32 + 3 * nt].reshape(nt, 3)
pub, done, cta = (tt[:, 0] - t0) / 1e3, (tt[:, 1] - t0) / 1e3, tt[:, 2] & 0xffffffff
smid = tt[:, 2] >> 32
exitt = (a[: 4 * n.value].reshape(-1, 4)[:, 3] - t0) / 1e3
print(f"{name} chi2 kernel {1e3 * ms:.1f} us, {nt} tiles, CTA exits min {np.nanmin(exitt):.1f} "
      f"median {np.median(exitt):.1f} max {np.nanmax(exitt):.1f} us")
order = np.argsort(done)
print("last 12 tiles done: tile, CTA, published us, done us, done - published, CTA's tiles, CTA exit")
for i in order[-12:]:
    k = int(cta[i])
    print(f"  {i:6d} {k:4d} {pub[i]:7.2f} {done[i]:7.2f} {done[i] - pub[i]:6.2f} "
          f"{int((cta == k).sum()):3d} {exitt[k]:7.2f}")
lat = done - pub
print(f"publish->fold per tile: median {np.median(lat):.2f} us, p90 {np.percentile(lat, 90):.2f}")
per = np.array([lat[cta == k].mean() for k in range(n.value)])
print("slowest CTAs by mean publish->fold (CTA, SM, us, tiles):",
      [(int(k), int(smid[cta == k][0]), round(float(per[k]), 2), int((cta == k).sum()))
       for k in np.argsort(per)[-6:]])
slow = int(np.argsort(per)[-1])
typ = int(np.argsort(per)[len(per) // 2])
for k, lab in ((slow, "slowest"), (typ, "typical")):
    idx = np.flatnonzero(cta == k)
    idx = idx[np.argsort(pub[idx])]
    print(f"{lab} CTA {k} (SM {int(smid[idx[0]])}): tile(pub,done) " +
          " ".join(f"{int(i)}({pub[i]:.1f},{done[i]:.1f})" for i in idx))
s2 = a[sms * 16: sms * 20].reshape(-1, 4)
print("stage-2 runs so far per CTA (slowest, typical):", int(s2[slow, 0]), int(s2[typ, 0]))
