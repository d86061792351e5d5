"""Randomised parity: random theory expressions over the reference grammar
(builtins, + - * /, unary minus, ^, exp/log/cos/sin/sqrt/pow, literals, p[m[k]],
f[m[k]]), random bindings, ragged datasets with t0 offsets and fit ranges.
The GPU objective (NVRTC-compiled per expression) must match the CPU oracle
within 1e-14 relative on totals and per-dataset values, give NaN exactly where
the oracle does, and raise the same exception type and message.  The
``logpow`` regime adds per-bin ``log``, per-bin-exponent ``pow`` / ``^`` and
``exp`` of bare ``t`` (theory.py:91-98, 450-452).
"""

import os
import numpy as np
import pytest

import paper_1604_02334_b200 as pkg
from conftest import rel
from oracle import musr_oracle as O
from paper_1604_02334_b200 import objective

pytestmark = pytest.mark.gpu
TOL = 1e-14   # "errors within 1e-9" needs <~1e-14 objective agreement
N_CASES = 40
# MUSR_FUZZ_SCALE=k runs k times as many cases per regime (deep runs; default 1)
SCALE = max(1, int(os.environ.get("MUSR_FUZZ_SCALE", "1")))


@pytest.fixture(autouse=True)
def _device(gpu_ok):
    yield
    objective.clear_cache()


def _uniform(rng, depth=0):
    """A parameter-only subexpression (small positive values)."""
    r = rng.random()
    if depth > 1 or r < 0.5:
        return f"p[m[{rng.integers(0, 6)}]]"
    if r < 0.7:
        return f"{rng.choice(['0.5', '2', '1e-1', '3.0'])} * p[m[{rng.integers(0, 6)}]]"
    if r < 0.85:
        return f"(p[m[{rng.integers(0, 6)}]] + f[m[{rng.integers(0, 2)}]])"
    return f"sqrt(p[m[{rng.integers(0, 6)}]])"


def _term(rng, depth=0):
    """A per-bin term of moderate magnitude on t in [0, 10] us."""
    r = rng.random()
    U = lambda: _uniform(rng, depth + 1)
    if depth > 2:
        r = r * 0.55
    if r < 0.10:
        return f"se(t, {U()})"
    if r < 0.20:
        return f"sg(t, {U()})"
    if r < 0.28:
        return f"stg(t, {U()})"
    if r < 0.36:
        return f"ge(t, {U()}, {rng.choice(['1.5', '0.5', '2', 'p[m[5]]'])})"
    if r < 0.46:
        return f"tf(t, {U()}, {U()})"
    if r < 0.52:
        return f"cos({U()} * t * t)"
    if r < 0.55:
        return f"exp(-{U()} * t)"
    if r < 0.65:
        return f"{_term(rng, depth + 1)} * {_term(rng, depth + 1)}"
    if r < 0.75:
        return f"({_term(rng, depth + 1)} + {_term(rng, depth + 1)})"
    if r < 0.80:
        return f"({_term(rng, depth + 1)} - 0.5 * {_term(rng, depth + 1)})"
    if r < 0.85:
        return f"{_term(rng, depth + 1)} / (1 + {U()})"
    if r < 0.90:
        return f"sin({U()} * t + {U()})"
    if r < 0.95:
        return f"(t / 10) ^ {rng.choice(['2', '0.5', '3', '1.5'])}"
    return f"-{_term(rng, depth + 1)}"


def _term_lp(rng, depth=0):
    """_term plus per-bin log, per-bin-exponent pow and exp(t)."""
    U = lambda: _uniform(rng, depth + 1)
    r = rng.random()
    if depth > 2 or r < 0.35:
        return _term(rng, depth)
    choices = [
        lambda: f"log(1 + {U()} * t)",
        lambda: f"log({U()} + t / 10)",
        lambda: f"log(se(t, {U()}) + {U()})",
        lambda: f"(1 + t / 10) ^ ({U()} * t)",
        lambda: f"pow({U()} + t / 10, sin(t))",
        lambda: f"(t / 10) ^ (t / 10)",
        lambda: f"{U()} ^ t",
        lambda: f"exp(t) / 100",
        lambda: f"exp(t / 10)",
        lambda: f"{_term_lp(rng, depth + 1)} * log(2 + t)",
        lambda: f"({_term_lp(rng, depth + 1)} + pow(1 + t, 0.5 * cos(t)))",
    ]
    return choices[int(rng.integers(0, len(choices)))]()


def _counts(rng, n, regime):
    """Counts: typical (Poisson 50-900), low (Poisson 0.2-5: many zero bins, MLH's
    d = 0 branch), or non-integer (the f64 data format)."""
    if regime == "low":
        return rng.poisson(rng.uniform(0.2, 5.0), n)
    if regime == "real":
        return rng.uniform(0.0, 300.0, n)
    return rng.poisson(rng.uniform(50, 900), n)


def _case(i, regime="typical"):
    rng = np.random.default_rng(1000 + i + (0 if regime == "typical" else 7919 * len(regime)))
    term = _term_lp if regime == "logpow" else _term
    src = f"p[m[0]] * ({term(rng)})"
    if rng.random() < 0.6:
        src += f" + p[m[1]] * ({term(rng, 1)})"
    expr = pkg.parse(src)
    dss = []
    for j in range(int(rng.integers(1, 4))):
        n = int(rng.choice([1, 777, 4096, 4097, 20000]))
        m = tuple(int(x) for x in rng.permutation(6))
        ds = pkg.MusrDataset(j, _counts(rng, n, regime), 10.0 / max(n, 100),
                             int(rng.integers(0, 4)) if n > 10 else 0, pkg.TheoryBinding(
                                 map=m, function_values=tuple(float(x) for x in rng.uniform(0, 1, 6))),
                             6, 7)
        if rng.random() < 0.3 and n > 10:
            ds.fit_range = (float(0.1 * ds.dt * n), float(0.8 * ds.dt * n))
        dss.append(ds)
    p = np.concatenate([rng.uniform(0.01, 0.5, 6), [rng.uniform(100, 1000), rng.uniform(1, 20)]])
    return src, expr, dss, p


CASES = [(i, "typical") for i in range(N_CASES * SCALE)] + [(i, "low") for i in range(10 * SCALE)] + \
        [(i, "real") for i in range(6 * SCALE)] + [(i, "logpow") for i in range(16 * SCALE)]


@pytest.mark.parametrize("i,regime", CASES)
def test_random_theories_match_oracle(i, regime):
    src, expr, dss, p = _case(i, regime)
    for kind in ("chi2", "mlh"):
        fn, ofn = (pkg.chi2, O.chi2) if kind == "chi2" else (pkg.mlh, O.mlh)
        try:
            per_o = []
            want = ofn(dss, expr, p, musr_error=pkg.MusrError, eval_error=pkg.EvalError,
                       per_dataset=per_o)
            want_exc = None
        except Exception as exc:  # noqa: BLE001  (reference exception semantics)
            want_exc = exc
        if want_exc is not None:
            with pytest.raises(type(want_exc)) as got:
                fn(dss, expr, p)
            assert str(got.value) == str(want_exc), (src, kind)
            continue
        got = fn(dss, expr, p)
        per = objective.session_for(dss, expr, pkg.TAU_MU_US, len(p), pkg.DeviceBackend()).per_dataset()
        if np.isnan(want):
            assert np.isnan(got), (src, kind)
            continue
        assert rel(got, want) <= TOL, (src, kind, got, want)
        for a, b in zip(per, per_o):
            assert (np.isnan(a) and np.isnan(b)) or rel(a, b) <= TOL, (src, kind, a, b)
