"""Pin the CPU oracle (oracle/musr_oracle.py) to the reference.

* bit-for-bit against the reference package itself on random problems
  (build container only, ``ref`` marker);
* against the committed golden vectors generated from the reference
  (tests/golden/make_golden.py), everywhere.  Golden values come from
  numpy's SIMD transcendentals on the build host; a different host CPU may
  differ in the last bit, so the tolerance is 1e-14 relative.
"""

import numpy as np
import pytest

from conftest import build_case, hexf, load_golden, rel
from oracle import musr_oracle as O
import paper_1604_02334_b200 as mirror
from paper_1604_02334_b200.theory import EvalError

META, ARR = load_golden()


def _oracle(kind, dss, expr, p, tau):
    fn = O.chi2 if kind == "chi2" else O.mlh
    per = []
    total = fn(dss, expr, p, tau, musr_error=mirror.MusrError, eval_error=EvalError,
               per_dataset=per)
    return total, per


@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
def test_oracle_matches_golden(case):
    dss, expr, p, tau = build_case(case, ARR, mirror)
    for kind, want in case["results"].items():
        if "error" in want:
            with pytest.raises(Exception) as exc:
                _oracle(kind, dss, expr, p, tau)
            assert type(exc.value).__name__ == want["error"]
            assert str(exc.value) == want["message"]
            continue
        total, per = _oracle(kind, dss, expr, p, tau)
        assert rel(total, hexf(want["value"])) <= 1e-14
        for a, b in zip(per, want["per_dataset"]):
            assert rel(a, hexf(b)) <= 1e-14


def test_pairwise_golden():
    for n in META["pairwise"]["lengths"]:
        x = ARR[f"pairwise/{n}"]
        assert O.pairwise_sum(x) == hexf(META["pairwise"]["sums"][str(n)])


@pytest.mark.ref
def test_oracle_bitwise_vs_reference(ref):
    """Random problems through both implementations: identical bits."""
    rng = np.random.default_rng(123)
    theories = ["p[m[0]] * se(t, p[m[1]])",
                "p[m[0]] * sg(t, p[m[1]]) * tf(t, p[m[2]] + f[m[0]], p[m[3]])",
                "p[m[0]] * stg(t, p[m[1]]) * se(t, p[m[2]]) + p[m[3]] * ge(t, p[m[4]], p[m[5]])",
                "pow(t + 1, p[m[0]]) - log(t + 2) * sin(t) + sqrt(t) / 7 + t ^ 2"]
    backend = ref.backend.Backend(1)
    for trial in range(12):
        src = theories[trial % len(theories)]
        expr_r = ref.theory.parse(src)
        dss = []
        for j in range(int(rng.integers(1, 4))):
            n = int(rng.integers(1, 3000))
            ds = ref.musr.MusrDataset(
                detector_index=j, counts=rng.integers(0, 500, n), dt=0.01 * rng.uniform(0.5, 2),
                t0_bin=int(rng.integers(0, 5)),
                binding=ref.theory.TheoryBinding(map=tuple(range(6)), function_values=(30.0,)),
                n0_slot=6, nbkg_slot=7)
            if rng.random() < 0.3:
                ds.fit_range = (rng.uniform(0, 3), rng.uniform(5, 30))
            dss.append(ds)
        p = np.concatenate([rng.uniform(0.05, 0.5, 6), [rng.uniform(100, 500), 10.0]])
        for kind in ("chi2", "mlh"):
            want = getattr(ref.musr, kind)(dss, expr_r, p, backend)
            got = getattr(O, kind)(dss, expr_r, p)
            assert got == want or (np.isnan(got) and np.isnan(want)), (src, kind)


@pytest.mark.ref
def test_oracle_pairwise_vs_reference(ref):
    rng = np.random.default_rng(7)
    for n in list(range(0, 70)) + [255, 256, 257, 4095, 4096, 4097, 100003]:
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 5)
        assert O.pairwise_sum(x) == ref.backend.pairwise_sum(x)


@pytest.mark.ref
def test_oracle_theory_values_vs_reference(ref):
    rng = np.random.default_rng(9)
    t = rng.uniform(0, 10, 5000)
    for src in ["p[m[0]] * sg(t,p[m[1]]) * tf(t,p[m[2]],f[m[3]]) - se(t, 0.3) ^ 2",
                "ge(t, p[m[0]], p[m[1]]) + stg(t, p[m[2]]) / (1 + exp(-t))",
                "-t ^ 2 + 2 ^ 3 ^ 0.5 * t"]:
        e = ref.theory.parse(src)
        b = ref.theory.TheoryBinding(map=(0, 1, 2, 3), function_values=(0.1, 0.2, 0.3, 0.4))
        p = rng.uniform(0.1, 2, 4)
        assert np.array_equal(O.evaluate(e, t, p, b), ref.theory.evaluate(e, t, p, b))
