"""Shared fixtures.  Markers: ``gpu`` (needs a B200 + libmusr_b200.so), ``ref``
(needs the reference package, present only in the build container)."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

# The reference package: its source tree in the build container, or the copy
# installed into the git-ignored baseline/_ref by tools/stage_reference.sh,
# which travels to the GPU host with the snapshot.
REF_SRC = next((d for d in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src"))
                if (d / "blk" / "musr.py").exists()), Path("/root/reference/pkg/src"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built libmusr_b200.so")
    config.addinivalue_line("markers", "ref: needs the reference package (baseline/_ref or "
                                       "/root/reference)")


def reference_available() -> bool:
    return (REF_SRC / "blk" / "musr.py").exists()


@pytest.fixture(scope="session")
def ref():
    """The reference package modules (blk.musr, blk.theory, blk.backend, blk.optimize)."""
    if not reference_available():
        pytest.skip("reference package not present (run tools/stage_reference.sh)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import blk.backend
    import blk.musr
    import blk.optimize
    import blk.theory

    class R:
        musr = blk.musr
        theory = blk.theory
        backend = blk.backend
        optimize = blk.optimize

    return R


def load_golden():
    meta = json.loads((GOLDEN / "musr_golden.json").read_text())
    arrays = dict(np.load(GOLDEN / "musr_golden.npz"))
    return meta, {k.replace("__", "/"): v for k, v in arrays.items()}


def hexf(s: str) -> float:
    return float.fromhex(s) if s != "nan" else float("nan")


def build_case(case, arrays, mirror):
    """Datasets/expr/p of a golden case built with the given package's types
    (``mirror`` = module providing MusrDataset/TheoryBinding/parse)."""
    dss = []
    for d in case["datasets"]:
        ds = mirror.MusrDataset(
            detector_index=d["detector_index"], counts=np.zeros(1), dt=hexf(d["dt"]),
            t0_bin=d["t0_bin"],
            binding=mirror.TheoryBinding(map=tuple(d["map"]),
                                         function_values=tuple(hexf(v) for v in d["f"])),
            n0_slot=d["n0_slot"], nbkg_slot=d["nbkg_slot"])
        ds.counts = arrays[d["counts"]].astype(np.float64)
        if d["fit_range"] is not None:
            ds.fit_range = (hexf(d["fit_range"][0]), hexf(d["fit_range"][1]))
        dss.append(ds)
    p = np.array([hexf(v) for v in case["p"]])
    return dss, mirror.parse(case["expr"]), p, hexf(case["tau_mu"])


# Largest relative difference seen by rel() in this session (GPU vs oracle /
# reference / golden), written to gpurun_out/parity_max_rel.json at the end.
PARITY = {"max_rel": 0.0, "where": None, "count": 0, "bitwise": 0}


def rel(a: float, b: float) -> float:
    if np.isnan(a) and np.isnan(b):
        r = 0.0
    elif a == b:
        r = 0.0
    else:
        r = abs(a - b) / max(abs(b), 1e-300)
    PARITY["count"] += 1
    PARITY["bitwise"] += int(r == 0.0)
    if r > PARITY["max_rel"]:
        import os

        PARITY["max_rel"] = float(r)
        PARITY["where"] = os.environ.get("PYTEST_CURRENT_TEST", "?")
    return r


def pytest_sessionfinish(session, exitstatus):
    if PARITY["count"] == 0:
        return
    out = ROOT / "gpurun_out"
    try:
        out.mkdir(exist_ok=True)
        (out / "parity_max_rel.json").write_text(json.dumps(PARITY, indent=1) + "\n")
    except OSError:
        pass


@pytest.fixture(scope="session")
def gpu_ok():
    """Skip unless a device and the library are available (GPU tests fail
    loudly instead when the library is missing on a GPU host)."""
    from paper_1604_02334_b200 import _lib

    lib = _lib.load()   # raises MusrDeviceError if the .so is missing
    if _lib.device_count() < 1:
        pytest.skip("no CUDA device")
    return lib
