"""CPU oracle for the uSR objective path -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm, used as the checker in
``tests/``, by ``__graft_entry__.smoke()`` and as the CPU baseline arm of
``bench.py``.  The product (``paper_1604_02334_b200``) never imports this.

Parity is pinned: ``tests/test_oracle.py`` checks this file bit-for-bit
against the reference package itself when it is importable (this build
container) and against golden vectors generated from it
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``).

Restated reference functions (paths under pkg/src/blk):

=====================================  ===========================================
oracle                                 reference
=====================================  ===========================================
times / errors / range_mask            musr.py:92-101
evaluate (stack machine over the AST)  theory.py:409-464, builtins theory.py:62-100
model_expected                         musr.py:150-162
pairwise_sum                           backend.py:79-95
map_reduce (fixed CHUNK, thread pool)  backend.py:24-27, 147-170, 174-207
chi2 / mlh                             musr.py:181-232
degrees_of_freedom                     musr.py:238-241
generate_synthetic / default_phases    musr.py:301-337
=====================================  ===========================================
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, List, Optional, Sequence

import numpy as np

CHUNK = 1 << 14                       # backend.py:27
TAU_MU_US = 2.197019                  # musr.py:48
GAMMA_MU = 2.0 * np.pi * 135.538809   # musr.py:49


class OracleMusrError(ValueError):
    """Stands in for blk.musr.MusrError."""


class OracleEvalError(ValueError):
    """Stands in for blk.theory.EvalError."""


# -- per-dataset accessors (musr.py:92-101) -----------------------------------------------

def times(ds) -> np.ndarray:
    return (np.arange(len(ds.counts)) - ds.t0_bin) * ds.dt


def errors(ds) -> np.ndarray:
    return np.maximum(1.0, np.sqrt(ds.counts))


def range_mask(ds) -> np.ndarray:
    t = times(ds)
    lo, hi = ds.fit_range if ds.fit_range is not None else (0.0, np.inf)
    return (t >= max(lo, 0.0)) & (t <= hi)


# -- theory interpreter (theory.py:62-100, 409-464) ---------------------------------------

def _builtin(name: str):
    if name == "se":
        return lambda t, lam: np.exp(-lam * t)
    if name == "ge":
        return lambda t, lam, beta: np.exp(-np.power(lam * t, beta))
    if name == "sg":
        return lambda t, sigma: np.exp(-0.5 * np.power(sigma * t, 2.0))
    if name == "stg":
        def stg(t, sigma):
            st2 = np.power(sigma * t, 2.0)
            return 1.0 / 3.0 + (2.0 / 3.0) * (1.0 - st2) * np.exp(-0.5 * st2)
        return stg
    if name == "tf":
        return lambda t, phi, nu: np.cos(2.0 * np.pi * nu * t + phi * np.pi / 180.0)
    return {"exp": np.exp, "log": np.log, "cos": np.cos, "sin": np.sin,
            "sqrt": np.sqrt, "pow": np.power}[name]


def _program(node, out: list) -> None:
    """Post-order instruction list; node classes are matched by name so ASTs
    of the reference package and of the product parser both work."""
    kind = type(node).__name__
    if kind == "Num":
        out.append(("num", node.value))
    elif kind == "TimeVar":
        out.append(("t",))
    elif kind == "SlotRef":
        out.append(("slot", node.array, node.slot))
    elif kind == "Unary":
        _program(node.operand, out)
        out.append(("neg",))
    elif kind == "Binary":
        _program(node.left, out)
        _program(node.right, out)
        out.append(("bin", node.op))
    elif kind == "Call":
        for a in node.args:
            _program(a, out)
        out.append(("call", node.name, len(node.args)))
    else:
        raise TypeError(f"unknown AST node {node!r}")


def evaluate(expr, t, p, binding, eval_error=OracleEvalError):
    p = np.asarray(p, dtype=np.float64)
    fv = np.asarray(binding.function_values, dtype=np.float64)
    m = binding.map
    scalar = np.isscalar(t) or np.ndim(t) == 0
    tv = np.float64(t) if scalar else np.asarray(t, dtype=np.float64)
    prog: list = []
    _program(expr.ast, prog)
    st: list = []
    for ins in prog:
        op = ins[0]
        if op == "num":
            st.append(ins[1])
        elif op == "t":
            st.append(tv)
        elif op == "slot":
            _, arr, k = ins
            if k >= len(m):
                raise eval_error(f"slot {k} not covered by map of length {len(m)}")
            j = m[k]
            src = p if arr == "p" else fv
            if j >= len(src):
                raise eval_error(
                    f"map entry m[{k}]={j} out of range for {arr!r} array of length {len(src)}")
            st.append(src[j])
        elif op == "neg":
            st.append(-st.pop())
        elif op == "bin":
            b = st.pop()
            a = st.pop()
            sym = ins[1]
            if sym == "+":
                st.append(a + b)
            elif sym == "-":
                st.append(a - b)
            elif sym == "*":
                st.append(a * b)
            elif sym == "/":
                st.append(a / b)
            else:
                st.append(np.power(a, b))
        else:
            _, name, argc = ins
            args = st[len(st) - argc:]
            del st[len(st) - argc:]
            st.append(_builtin(name)(*args))
    (res,) = st
    return float(res) if scalar else np.asarray(res, dtype=np.float64)


def model_expected(ds, expr, p, tau_mu: float = TAU_MU_US, eval_error=OracleEvalError):
    t = times(ds)
    a = evaluate(expr, t, p, ds.binding, eval_error)
    return p[ds.n0_slot] * np.exp(-t / tau_mu) * (1.0 + a) + p[ds.nbkg_slot]


# -- reduction (backend.py:79-95, 157-207) ---------------------------------------------------

def pairwise_sum(terms) -> float:
    x = np.asarray(terms, dtype=np.float64)
    if x.size == 0:
        return 0.0
    while x.size > 1:
        even = x[0:x.size - (x.size & 1):2] + x[1::2][: x.size // 2]
        x = np.concatenate([even, x[-1:]]) if x.size & 1 else even
    return float(x[0])


_POOLS = {}


def map_reduce(fn: Callable, *arrays, workers: int = 1) -> float:
    n = len(arrays[0])
    if n == 0:
        return 0.0
    bounds = [(lo, min(lo + CHUNK, n)) for lo in range(0, n, CHUNK)]
    job = lambda b: np.asarray(fn(*[a[b[0]:b[1]] for a in arrays]), dtype=np.float64)
    if workers > 1 and len(bounds) > 1:
        pool = _POOLS.get(workers)
        if pool is None:
            pool = _POOLS[workers] = ThreadPoolExecutor(max_workers=workers)
        parts = list(pool.map(job, bounds))
    else:
        parts = [job(b) for b in bounds]
    return pairwise_sum(parts[0] if len(parts) == 1 else np.concatenate(parts))


# -- objectives (musr.py:181-241) ------------------------------------------------------------

def _chi2_terms(dd, mm, ee):
    return ((dd - mm) / ee) ** 2


def _mlh_terms(dd, mm):
    with np.errstate(divide="ignore", invalid="ignore"):
        lt = np.where(dd > 0, dd * np.log(np.where(dd > 0, dd, 1.0) / mm), 0.0)
    return 2.0 * ((mm - dd) + lt)


def chi2(datasets, expr, p, tau_mu: float = TAU_MU_US, workers: int = 1,
         musr_error=OracleMusrError, eval_error=OracleEvalError, per_dataset: list = None):
    p = np.asarray(p, dtype=np.float64)
    total = 0.0
    for ds in datasets:
        mask = range_mask(ds)
        if not mask.any():
            raise musr_error(f"detector {ds.detector_index}: empty fit range")
        model = model_expected(ds, expr, p, tau_mu, eval_error)[mask]
        s = map_reduce(_chi2_terms, ds.counts[mask], model, errors(ds)[mask], workers=workers)
        if per_dataset is not None:
            per_dataset.append(s)
        total += s
    return total


def mlh(datasets, expr, p, tau_mu: float = TAU_MU_US, workers: int = 1,
        musr_error=OracleMusrError, eval_error=OracleEvalError, per_dataset: list = None):
    p = np.asarray(p, dtype=np.float64)
    total = 0.0
    for ds in datasets:
        mask = range_mask(ds)
        if not mask.any():
            raise musr_error(f"detector {ds.detector_index}: empty fit range")
        model = model_expected(ds, expr, p, tau_mu, eval_error)[mask]
        nonpos = model <= 0
        if np.any(nonpos):
            bad = int(np.flatnonzero(mask)[np.argmax(nonpos)])
            raise musr_error(f"detector {ds.detector_index}: model is non-positive at bin {bad}")
        s = map_reduce(_mlh_terms, ds.counts[mask], model, workers=workers)
        if per_dataset is not None:
            per_dataset.append(s)
        total += s
    return total


def degrees_of_freedom(datasets, fixed) -> int:
    return sum(int(range_mask(ds).sum()) for ds in datasets) - int((~np.asarray(fixed)).sum())


# -- synthetic data (musr.py:301-337) --------------------------------------------------------

def default_phases(n: int = 16) -> np.ndarray:
    return np.arange(n) * (360.0 / n)


def generate_synthetic(make_dataset, truth_values, expr, bindings, n0_slots, nbkg_slots,
                       nbins: int, dt: float, seed: int, t0_bin: int = 0,
                       tau_mu: float = TAU_MU_US) -> List:
    """Poisson histograms, one per binding, from one default_rng(seed) in
    detector order.  ``make_dataset(j, counts, dt, t0_bin, binding, n0, nbkg)``
    builds the dataset object of whichever package is under test."""
    rng = np.random.default_rng(seed)
    truth = np.asarray(truth_values, dtype=np.float64)
    out = []
    for j, b in enumerate(bindings):
        ds = make_dataset(j, np.zeros(nbins, dtype=np.int64), dt, t0_bin, b,
                          n0_slots[j], nbkg_slots[j])
        lam = model_expected(ds, expr, truth, tau_mu)
        if np.any(lam < 0):
            raise OracleMusrError(
                f"detector {j}: negative expected count at bin {int(np.argmax(lam < 0))}")
        ds.counts = rng.poisson(lam).astype(np.float64)
        out.append(ds)
    return out


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
