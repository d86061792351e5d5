"""Native muSR data file reader/writer (csrc/musr_io.cpp, musrio.py) against
the reference's load_musr_data / store_musr_data (io.py:109-212).

CPU only: the loader is host code in libmusr_b200.so (no device needed).
Parity is pinned two ways: live against the reference (``ref`` fixture, build
container) and against committed golden outcomes (tests/golden/io_cases.json,
made by tests/golden/make_golden_io.py from the reference).
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import musrio

GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLDEN))
from io_corpus import CASES  # noqa: E402  (shared with make_golden_io.py)


def _outcome(load, path):
    """('ok', [dataset summaries]) or ('error', type name, message with the
    path replaced by {path})."""
    try:
        dss = load(path)
    except Exception as exc:  # noqa: BLE001 - we compare exception types
        return ["error", type(exc).__name__, str(exc).replace(str(path), "{path}")]
    return ["ok", [[int(d.detector_index), float(d.dt).hex(), int(d.t0_bin), int(d.n0_slot),
                    int(d.nbkg_slot), [int(x) for x in d.binding.map],
                    [float(x).hex() for x in d.binding.function_values],
                    [float(x).hex() for x in np.asarray(d.counts, dtype=np.float64)]]
                   for d in dss]]


def _write(tmp_path, name, content):
    p = tmp_path / f"{name}.musr"
    p.write_bytes(content.encode("utf-8") if isinstance(content, str) else content)
    return p


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("threads", [1, 3])
def test_loader_matches_golden(tmp_path, name, threads):
    want = json.loads((GOLDEN / "io_cases.json").read_text())[name]
    p = _write(tmp_path, name, CASES[name])
    got = _outcome(lambda q: musrio.load_musr_data(q, n_threads=threads), p)
    assert got == want


@pytest.mark.parametrize("name", sorted(CASES))
def test_loader_matches_reference_live(ref, tmp_path, name):
    import blk.io

    p = _write(tmp_path, name, CASES[name])
    assert _outcome(musrio.load_musr_data, p) == _outcome(blk.io.load_musr_data, p)


def _random_datasets(rng, n, nbins_max=3000):
    out = []
    for j in range(n):
        nb = int(rng.integers(1, nbins_max))
        counts = rng.poisson(rng.uniform(1, 5000), nb).astype(np.float64)
        out.append(pkg.MusrDataset(
            detector_index=j * 3 - 2, counts=counts, dt=float(rng.choice([0.001, 1e-5, 0.1 + 0.2, 7.0, 1e16])),
            t0_bin=int(rng.integers(-5, 50)),
            binding=pkg.TheoryBinding(map=tuple(int(x) for x in rng.integers(0, 9, rng.integers(0, 6))),
                                      function_values=tuple(rng.standard_normal(rng.integers(0, 3)) * 100)),
            n0_slot=int(rng.integers(0, 8)), nbkg_slot=int(rng.integers(0, 8))))
    return out


def test_writer_byte_identical_to_reference(ref, tmp_path):
    import blk.io

    rng = np.random.default_rng(0)
    dss = _random_datasets(rng, 7)
    dss[2].counts = np.array([0.0, 3.9, 1e6, 17.0] * 9)          # truncation like astype(int64)
    a, b = tmp_path / "ours.musr", tmp_path / "ref.musr"
    musrio.store_musr_data(a, dss, n_threads=4)
    blk.io.store_musr_data(b, dss)
    assert a.read_bytes() == b.read_bytes()
    musrio.store_musr_data(a, [], n_threads=2)
    blk.io.store_musr_data(b, [])
    assert a.read_bytes() == b.read_bytes()


def test_round_trip_large_multithreaded(tmp_path):
    """Several MB of counts, written and read back with 8 threads."""
    rng = np.random.default_rng(1)
    dss = _random_datasets(rng, 6, nbins_max=400_000)
    p = tmp_path / "big.musr"
    musrio.store_musr_data(p, dss, n_threads=8)
    back = musrio.load_musr_data(p, n_threads=8)
    assert len(back) == len(dss)
    for x, y in zip(back, dss):
        assert np.array_equal(x.counts, np.trunc(y.counts))
        assert (x.detector_index, x.dt, x.t0_bin, x.n0_slot, x.nbkg_slot) == \
            (y.detector_index, y.dt, y.t0_bin, y.n0_slot, y.nbkg_slot)
        assert x.binding == y.binding
    # the same file with an error late in it: the error (not a block before it) is reported
    text = p.read_text().splitlines()
    text[len(text) - 40] = "  12 x 13"
    bad = tmp_path / "bad.musr"
    bad.write_text("\n".join(text))
    with pytest.raises(musrio.FormatError, match=f":{len(text) - 39}: malformed line: '12 x 13'"):
        musrio.load_musr_data(bad, n_threads=8)


def test_missing_file_raises_oserror(tmp_path):
    with pytest.raises(FileNotFoundError):
        musrio.load_musr_data(tmp_path / "nope.musr")
