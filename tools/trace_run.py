"""Per-CTA timeline of one objective launch (developer tool, MUSR_TRACE=1)."""
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
for kind in (0, 1):
    (musr.chi2 if kind == 0 else musr.mlh)(ds, w.expr, w.params)
    ms = s.time_evals(kind, 3, 1, int(os.environ.get("MUSR_FLUSH", "1"))) / 3
    buf = (C.c_uint64 * (4 * 4096))()
    n = C.c_int()
    _lib.check(s._lib.musr_debug_trace(s._handle, kind, buf, len(buf), C.byref(n)), s._handle, "trace")
    t = np.array(buf[: 4 * n.value], dtype=np.int64).reshape(-1, 4).astype(float)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    rel[t == 0] = np.nan
    print(f"{name} kind={kind} kernel {1e3*ms:.1f} us, {n.value} CTAs")
    tiles = np.array(buf[: 4 * n.value], dtype=np.int64).reshape(-1, 4)[:, 2]
    ex = rel[:, 3]
    order = np.argsort(ex)
    print("  tiles/CTA min %d max %d; 10 latest CTAs (exit us, tiles): %s" % (
        tiles.min(), tiles.max(), [(round(ex[i], 1), int(tiles[i])) for i in order[-10:]]))
    print("  10 earliest: %s" % [(round(ex[i], 1), int(tiles[i])) for i in order[:10]])
    ext = np.array(buf[4 * n.value: 8 * n.value], dtype=np.int64).reshape(-1, 4).astype(float)
    ext_rel = (ext - t0) / 1e3
    ext_rel[ext == 0] = np.nan
    cols = [("start", rel[:, 0]), ("rows done", ext_rel[:, 0]), ("rows barrier", ext_rel[:, 1]),
            ("after prologue", rel[:, 1]), ("1st data", ext_rel[:, 2]), ("1st tile done", ext_rel[:, 3]),
            ("producer exit", rel[:, 3])]
    prod = np.array(buf[8 * n.value: 16 * n.value], dtype=np.int64).reshape(-1, 8).astype(float)
    tiles_cta = tiles.astype(float)
    names = ["wait idx", "wait done", "fold", "grab", "publish", "rest", "tma", "grab-ahead"]
    tot = prod.sum(axis=1)
    print("  producer cycles per tile (median over CTAs): " + ", ".join(
        f"{nm} {np.median(prod[:, k] / np.maximum(tiles_cta, 1)):.0f}" for k, nm in enumerate(names)) +
        f"; total {np.median(tot / np.maximum(tiles_cta, 1)):.0f}")
    s2 = np.array(buf[16 * n.value: 20 * n.value], dtype=np.int64).reshape(-1, 4)
    has = s2[:, 2] > 0
    if has.any():
        rel2 = (s2[has, 1:].astype(float) - t0) / 1e3
        order2 = np.argsort(rel2[:, 2])[-4:]
        print("  latest stage-2 runs (check, start, end us; CTA exit us): " + "; ".join(
            f"{rel2[i, 0]:.1f} {rel2[i, 1]:.1f} {rel2[i, 2]:.1f} (exit {ex[np.flatnonzero(has)[i]]:.1f})"
            for i in order2))
    for label, v in cols:
        v = v[~np.isnan(v)]
        if len(v):
            print(f"  {label:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us  (n={len(v)})")
