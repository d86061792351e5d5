"""muSR data file ingest: native loader/writer vs the reference's Python
(io.py:124-212) on a synthetic C-shaped file (developer tool; the reference
arm needs /root/reference, i.e. the build container)."""
import sys, time, tempfile, os, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import musrio, workloads as W

n_hist = int(sys.argv[1]) if len(sys.argv) > 1 else 8
nbins = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
w = W.c4(n_hist=n_hist, nbins=nbins)
dss = W.synthesize(w)
out = {"datasets": n_hist, "bins": n_hist * nbins, "threads": os.cpu_count()}
with tempfile.TemporaryDirectory() as d:
    p = Path(d) / "c.musr"
    t0 = time.perf_counter(); musrio.store_musr_data(p, dss); out["native_store_s"] = time.perf_counter() - t0
    out["file_mb"] = p.stat().st_size / 1e6
    t0 = time.perf_counter(); back = musrio.load_musr_data(p); out["native_load_s"] = time.perf_counter() - t0
    assert all(np.array_equal(a.counts, b.counts) for a, b in zip(back, dss))
    ref = Path("/root/reference/pkg/src")
    if ref.exists():
        sys.path.insert(0, str(ref))
        import blk.io
        q = Path(d) / "r.musr"
        t0 = time.perf_counter(); blk.io.store_musr_data(q, dss); out["ref_store_s"] = time.perf_counter() - t0
        assert p.read_bytes() == q.read_bytes()
        t0 = time.perf_counter(); rb = blk.io.load_musr_data(q); out["ref_load_s"] = time.perf_counter() - t0
        assert all(np.array_equal(a.counts, b.counts) for a, b in zip(back, rb))
        out["load_speedup"] = out["ref_load_s"] / out["native_load_s"]
        out["store_speedup"] = out["ref_store_s"] / out["native_store_s"]
print(json.dumps(out))
