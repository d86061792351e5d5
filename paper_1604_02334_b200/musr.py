"""uSR objective API -- drop-in mirror of ``pkg/src/blk/musr.py`` backed by the GPU.

Same names, signatures, argument meaning and exceptions as the reference:

* ``PhysicsConstants``, ``MusrError``, ``MusrDataset``, ``ParameterSet``,
  ``FitResult``                                            musr.py:47-145
* ``chi2``, ``mlh`` -- evaluated by libmusr_b200.so        musr.py:181-232
* ``OBJECTIVES`` registry read by ``minimize``             musr.py:235, 261-263
* ``degrees_of_freedom``                                   musr.py:238-241
* ``minimize`` -- the reference fit driver over the restated Nelder-Mead
                                                           musr.py:246-296
* ``default_phases``                                       musr.py:335-337

``chi2``/``mlh`` accept the reference's own ``MusrDataset``/``TheoryExpr``
objects as well as these mirrors (duck typing), so
``install(blk.musr)`` makes the reference's own fit loop and CLI run on B200.
The ``backend`` argument selects the GPU (``DeviceBackend``); any other object
(e.g. the reference's CPU ``Backend``) means device 0.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import objective as _obj
from ._lib import KIND_CHI2, KIND_MLH
from .objective import DeviceBackend
from .optimize import MinimizeConfig, nelder_mead
from .theory import TheoryBinding, TheoryExpr

__all__ = [
    "PhysicsConstants",
    "MusrDataset",
    "ParameterSet",
    "FitResult",
    "MusrError",
    "chi2",
    "mlh",
    "chi2_batch",
    "mlh_batch",
    "OBJECTIVES",
    "OBJECTIVES_BATCH",
    "degrees_of_freedom",
    "minimize",
    "default_phases",
    "install",
    "uninstall",
    "TAU_MU_US",
    "GAMMA_MU",
]

TAU_MU_US = 2.197019                     # musr.py:48
GAMMA_MU = 2.0 * np.pi * 135.538809     # musr.py:49


@dataclass(frozen=True)
class PhysicsConstants:
    tau_mu: float = TAU_MU_US
    gamma_mu: float = GAMMA_MU

    def __post_init__(self):
        if self.tau_mu <= 0:
            raise ValueError("tau_mu must be positive")


class MusrError(ValueError):
    pass


_obj.ERRORS.musr = MusrError


@dataclass
class MusrDataset:
    """One detector histogram plus its theory binding (musr.py:66-101)."""

    detector_index: int
    counts: np.ndarray
    dt: float
    t0_bin: int
    binding: TheoryBinding
    n0_slot: int
    nbkg_slot: int
    fit_range: Optional[tuple] = None

    def __setattr__(self, name, value):
        # any field assignment invalidates the session cache's O(1) check
        _obj.DATASET_MUTATIONS[0] += 1
        object.__setattr__(self, name, value)

    def __post_init__(self):
        self.counts = np.asarray(self.counts)
        j = self.detector_index
        if len(self.counts) < 1:
            raise MusrError(f"detector {j}: empty histogram")
        if self.dt <= 0:
            raise MusrError(f"detector {j}: dt must be positive")
        neg = self.counts < 0
        if np.any(neg):
            raise MusrError(f"detector {j}: negative count at bin {int(np.argmax(neg))}")
        self.counts = self.counts.astype(np.float64)

    # Host-side accessors with the reference semantics (used at session build
    # and by degrees_of_freedom; never per evaluation).
    def times(self) -> np.ndarray:
        return (np.arange(len(self.counts)) - self.t0_bin) * self.dt

    def errors(self) -> np.ndarray:
        return np.maximum(1.0, np.sqrt(self.counts))

    def range_mask(self) -> np.ndarray:
        t = self.times()
        lo, hi = self.fit_range if self.fit_range is not None else (0.0, np.inf)
        return (t >= max(lo, 0.0)) & (t <= hi)


@dataclass
class ParameterSet:
    """Full parameter vector with names, steps, bounds, fixed flags (musr.py:104-136)."""

    values: np.ndarray
    names: list
    step_sizes: np.ndarray
    bounds: Optional[list] = None
    fixed: Optional[np.ndarray] = None

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)
        self.step_sizes = np.asarray(self.step_sizes, dtype=np.float64)
        n = len(self.values)
        if len(self.names) != n or len(self.step_sizes) != n:
            raise MusrError("values, names and step_sizes must have equal lengths")
        if self.bounds is None:
            self.bounds = [None] * n
        if self.fixed is None:
            self.fixed = np.zeros(n, dtype=bool)
        self.fixed = np.asarray(self.fixed, dtype=bool)

    def copy_with(self, values: np.ndarray) -> "ParameterSet":
        return ParameterSet(
            values=np.asarray(values, dtype=np.float64).copy(),
            names=list(self.names),
            step_sizes=self.step_sizes.copy(),
            bounds=list(self.bounds),
            fixed=self.fixed.copy(),
        )

    def slot(self, name: str) -> int:
        return self.names.index(name)


@dataclass
class FitResult:
    best_parameters: ParameterSet
    objective_value: float
    iterations: int
    objective_evaluations: int
    converged: bool


# -- objectives (GPU) ------------------------------------------------------------------

_DEFAULT_BACKEND = DeviceBackend()


def _device_backend(backend) -> DeviceBackend:
    return backend if isinstance(backend, DeviceBackend) else _DEFAULT_BACKEND


def _evaluate(kind: int, datasets, expr, p, backend, constants) -> float:
    # the same problem as the last call: validated and launched in C (musr_pyfast.c)
    v = _obj.fast_evaluate(kind, datasets, expr, p, backend, constants)
    if v is not None:
        return v
    p = np.asarray(p, dtype=np.float64)
    if len(datasets) == 0:
        return 0.0
    sess = _obj.session_for(datasets, expr, float(constants.tau_mu), len(p),
                            _device_backend(backend))
    v = sess.evaluate(kind, p)
    _obj.fast_remember(sess, datasets, expr, backend, constants)
    return v


def chi2(
    datasets: Sequence,
    expr: TheoryExpr,
    p: np.ndarray,
    backend=None,
    constants: PhysicsConstants = PhysicsConstants(),
) -> float:
    """Sum over datasets and in-range bins of ((d - N) / max(1, sqrt(d)))^2,
    evaluated on the GPU (musr.py:181-201)."""
    return _evaluate(KIND_CHI2, datasets, expr, p, backend, constants)


def mlh(
    datasets: Sequence,
    expr: TheoryExpr,
    p: np.ndarray,
    backend=None,
    constants: PhysicsConstants = PhysicsConstants(),
) -> float:
    """2 * sum of (N - d) + d*log(d/N), evaluated on the GPU (musr.py:204-232)."""
    return _evaluate(KIND_MLH, datasets, expr, p, backend, constants)


OBJECTIVES = {"chi2": chi2, "mlh": mlh}


def _evaluate_batch(kind: int, datasets, expr, P, backend, constants) -> np.ndarray:
    P = np.asarray(P, dtype=np.float64)
    if P.ndim != 2:
        raise ValueError("P must be a 2-D array: one parameter vector per row")
    if len(datasets) == 0:
        return np.zeros(P.shape[0], dtype=np.float64)
    sess = _obj.session_for(datasets, expr, float(constants.tau_mu), P.shape[1],
                            _device_backend(backend))
    return sess.evaluate_batch(kind, P)


def chi2_batch(datasets: Sequence, expr: TheoryExpr, P: np.ndarray, backend=None,
               constants: PhysicsConstants = PhysicsConstants()) -> np.ndarray:
    """chi2 at every row of P (n_points x n_p) in one pass over the histograms
    per 8 points; element i is bit-identical to ``chi2(datasets, expr, P[i])``
    and the first failing row raises its exception."""
    return _evaluate_batch(KIND_CHI2, datasets, expr, P, backend, constants)


def mlh_batch(datasets: Sequence, expr: TheoryExpr, P: np.ndarray, backend=None,
              constants: PhysicsConstants = PhysicsConstants()) -> np.ndarray:
    """mlh at every row of P; see chi2_batch."""
    return _evaluate_batch(KIND_MLH, datasets, expr, P, backend, constants)


OBJECTIVES_BATCH = {"chi2": chi2_batch, "mlh": mlh_batch}
# batching is used by minimize only while the registry entry is still this
# package's own objective (a user-replaced OBJECTIVES entry runs unbatched)
OBJECTIVES_BATCH_OF = {"chi2": chi2, "mlh": mlh}


def degrees_of_freedom(datasets: Sequence, params: ParameterSet) -> int:
    nbins = sum(int(ds.range_mask().sum()) for ds in datasets)
    return nbins - int((~np.asarray(params.fixed)).sum())


# -- fit driver (reference loop, musr.py:246-296) ----------------------------------------

def minimize(
    objective: str,
    datasets: Sequence,
    expr: TheoryExpr,
    params: ParameterSet,
    backend=None,
    constants: PhysicsConstants = PhysicsConstants(),
    config: Optional[MinimizeConfig] = None,
    objective_fn=None,
) -> FitResult:
    batch_fn = None
    if objective_fn is None:
        obj = OBJECTIVES[objective]

        def objective_fn(p):
            return obj(datasets, expr, p, backend, constants)

        objb = OBJECTIVES_BATCH.get(objective) if obj is OBJECTIVES_BATCH_OF.get(objective) \
            else None
        if objb is not None:
            def batch_fn(P):   # simplex / shrink points in one pass (bit-identical values)
                return objb(datasets, expr, P, backend, constants)

    free = np.flatnonzero(~params.fixed)
    full = params.values.copy()
    if len(free) == 0:
        value = float(objective_fn(full))
        return FitResult(params.copy_with(full), value, 0, 1, True)

    steps = params.step_sizes[free]
    if np.any(steps <= 0):
        raise MusrError("free parameters need positive step sizes")
    box = [params.bounds[k] or (-np.inf, np.inf) for k in free]
    lo = np.array([b[0] for b in box], dtype=np.float64)
    hi = np.array([b[1] for b in box], dtype=np.float64)

    def reduced(x: np.ndarray) -> float:
        full[free] = x
        return float(objective_fn(full))

    reduced_batch = None
    if batch_fn is not None:
        def reduced_batch(X: np.ndarray) -> np.ndarray:
            P = np.repeat(full[None, :], len(X), axis=0)
            P[:, free] = X
            return batch_fn(P)

    if batch_fn is not None and len(datasets) > 0:
        # Built-in objective: the whole loop runs natively (musr_minimize, the
        # same iterates bit for bit); only the start is evaluated here, so the
        # reference's errors are raised exactly where nelder_mead raises them.
        return _minimize_native(objective, datasets, expr, params, backend, constants, config,
                                free, full, steps, lo, hi, reduced)
    res = nelder_mead(reduced, params.values[free], steps, lo, hi, config, reduced_batch)
    full[free] = res.x
    return FitResult(params.copy_with(full), res.fun, res.iterations, res.evaluations,
                     res.converged)


def _minimize_native(objective, datasets, expr, params, backend, constants, config, free, full,
                     steps, lo, hi, reduced) -> FitResult:
    import ctypes as C

    from ._lib import check as _check
    from .optimize import OptimizeError

    cfg = config or MinimizeConfig()
    x0 = np.minimum(np.maximum(np.asarray(params.values[free], dtype=np.float64), lo), hi)
    first = reduced(x0)                    # optimize.py:81-83 (static errors raise here)
    if not np.isfinite(first):
        raise OptimizeError(f"objective is not finite at the initial point ({first})")
    full[free] = x0
    sess = _obj.session_for(datasets, expr, float(constants.tau_mu), len(full),
                            _device_backend(backend))
    n = len(free)
    kind = KIND_CHI2 if objective == "chi2" else KIND_MLH
    dp = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    pf, x0c, st, lo_, hi_ = dp(full), dp(x0), dp(steps), dp(lo), dp(hi)
    idx = np.ascontiguousarray(free, dtype=np.int32)
    best, fail = np.zeros(n), np.zeros(n)
    bf, it, ev, conv = C.c_double(), C.c_int64(), C.c_int64(), C.c_int()
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    rc = sess._lib.musr_minimize(sess._handle, kind, P(pf), len(pf),
                                 idx.ctypes.data_as(C.POINTER(C.c_int32)), n, P(x0c), first, P(st),
                                 P(lo_), P(hi_), cfg.tol_f, cfg.max_evaluations or 400 * n,
                                 cfg.restarts, P(best), C.byref(bf), C.byref(it), C.byref(ev),
                                 C.byref(conv), P(fail))
    if rc == 100:                          # MUSR_NM_RAISED: re-evaluate there, raising as the reference
        reduced(fail)
        raise RuntimeError("native Nelder-Mead reported an error the objective did not raise")
    _check(rc, sess._handle, "musr_minimize")
    full[free] = best
    return FitResult(params.copy_with(full), bf.value, it.value, ev.value, bool(conv.value))


def default_phases(n_detectors: int = 16) -> np.ndarray:
    """phi_j = j * 360 / n degrees (musr.py:335-337)."""
    return np.arange(n_detectors) * (360.0 / n_detectors)


# -- integration into the reference package --------------------------------------------

def install(musr_module, theory_module=None, backend: Optional[DeviceBackend] = None):
    """Route a host package's objective registry to the GPU.

    ``install(blk.musr, blk.theory)`` replaces ``blk.musr.OBJECTIVES["chi2"/"mlh"]``
    (read at call time by ``blk.musr.minimize``, musr.py:261-263) with GPU
    objectives raising the host package's ``MusrError``/``EvalError``.  Returns
    the previous registry entries so callers can restore them.
    """
    previous = dict(musr_module.OBJECTIVES)
    _obj.ERRORS.musr = getattr(musr_module, "MusrError", MusrError)
    if theory_module is not None and hasattr(theory_module, "EvalError"):
        _obj.ERRORS.eval = theory_module.EvalError
    forced = backend

    def gpu_chi2(datasets, expr, p, backend=None, constants=musr_module.PhysicsConstants()):
        return chi2(datasets, expr, p, forced or backend, constants)

    def gpu_mlh(datasets, expr, p, backend=None, constants=musr_module.PhysicsConstants()):
        return mlh(datasets, expr, p, forced or backend, constants)

    musr_module.OBJECTIVES["chi2"] = gpu_chi2
    musr_module.OBJECTIVES["mlh"] = gpu_mlh
    _obj.clear_cache()
    return previous


def uninstall(musr_module, previous) -> None:
    """Undo ``install``: restore the registry entries it returned and this
    package's own exception classes."""
    musr_module.OBJECTIVES.clear()
    musr_module.OBJECTIVES.update(previous)
    _obj.ERRORS.musr = MusrError
    from .theory import EvalError

    _obj.ERRORS.eval = EvalError
    _obj.clear_cache()
