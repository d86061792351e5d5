"""CPU tests of the drop-in call's C fast path (csrc/musr_pyfast.c).

The module's hit/miss logic is exercised with a stand-in for musr_eval (a
ctypes callback that writes a recognisable total), so every invalidation rule
is checked without a GPU: the remembered problem must be answered only while
the call is provably the same as the one the session was built from, exactly
as the Python path (objective.session_for) decides.  The GPU tests run the
real path (tests/test_gpu.py)."""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np
import pytest

from paper_1604_02334_b200 import _lib

EVAL_T = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                     C.c_void_p, C.c_void_p)


@dataclass
class _DS:                         # shaped like the reference's MusrDataset (musr.py:66-90)
    detector_index: int
    counts: np.ndarray
    dt: float = 0.01


class _Slotted:
    __slots__ = ("counts",)

    def __init__(self, counts):
        self.counts = counts


class _Sess:
    pass


@pytest.fixture
def fast():
    """The module bound to a fake musr_eval: total = sum(p) + 1000 * kind;
    status and the first bad bin are settable; calls are counted."""
    from paper_1604_02334_b200 import _pyfast as mod

    state = {"calls": 0, "rc": 0, "bad": -1}

    def fake(ctx, kind, p, n_p, sums, bad, total):
        state["calls"] += 1
        pv = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), (n_p,))
        C.cast(total, C.POINTER(C.c_double))[0] = float(pv.sum()) + 1000.0 * kind
        C.cast(bad, C.POINTER(C.c_int64))[0] = state["bad"]
        return state["rc"]

    cb = EVAL_T(fake)
    mod.init(C.cast(cb, C.c_void_p).value, np.ndarray, np.dtype(np.float64))
    state["mod"] = mod
    yield state
    mod.forget()
    _lib._PYFAST = None            # the next real use re-binds the library's musr_eval
    del cb


def _problem(n=3):
    dss = [_DS(j, np.arange(5.0) + j) for j in range(n)]
    for d in dss:
        d.counts.flags.writeable = False          # what _FrozenCounts does
    sess = _Sess()
    sess.lock = threading.Lock()
    sess.sums = np.zeros(n)
    sess.bad = np.full(n, -1, dtype=np.int64)
    sess.total = np.zeros(1)
    expr, backend, consts = object(), object(), object()
    return dss, sess, expr, backend, consts


def _remember(mod, dss, sess, expr, backend, consts, n_p=3):
    return mod.remember(sess, dss, expr, backend, consts, tuple(d.counts for d in dss), 1, n_p,
                        len(dss), sess.sums.ctypes.data, sess.bad.ctypes.data,
                        sess.total.ctypes.data, sess.lock)


def test_hit_returns_device_total_and_misses_on_foreign_arguments(fast):
    mod = fast["mod"]
    dss, sess, expr, be, cs = _problem()
    assert _remember(mod, dss, sess, expr, be, cs)
    p = np.array([1.0, 2.0, 3.0])
    assert mod.evaluate(0, dss, expr, p, be, cs) == 6.0
    assert mod.evaluate(1, dss, expr, p, be, cs) == 1006.0
    assert fast["calls"] == 2
    # anything not provably the remembered problem goes to the Python path
    assert mod.evaluate(0, list(dss), expr, p, be, cs) is None        # another list object
    assert mod.evaluate(0, dss, object(), p, be, cs) is None          # theory
    assert mod.evaluate(0, dss, expr, p, None, cs) is None            # backend
    assert mod.evaluate(0, dss, expr, p, be, object()) is None        # constants
    assert mod.evaluate(2, dss, expr, p, be, cs) is None              # unknown kind
    assert mod.evaluate(0, dss, expr, [1.0, 2.0, 3.0], be, cs) is None          # not an ndarray
    assert mod.evaluate(0, dss, expr, p.astype(np.float32), be, cs) is None     # dtype
    assert mod.evaluate(0, dss, expr, p.astype(">f8"), be, cs) is None          # byte order
    assert mod.evaluate(0, dss, expr, np.zeros(4), be, cs) is None              # length
    assert mod.evaluate(0, dss, expr, np.zeros(6)[::2], be, cs) is None         # strided
    assert mod.evaluate(0, dss, expr, np.zeros((1, 3)), be, cs) is None         # 2-D
    assert fast["calls"] == 2


def test_list_edits_and_attribute_assignment_invalidate(fast):
    mod = fast["mod"]
    p = np.ones(3)
    dss, sess, expr, be, cs = _problem()
    _remember(mod, dss, sess, expr, be, cs)
    d = dss.pop()
    assert mod.evaluate(0, dss, expr, p, be, cs) is None              # shorter list
    dss.append(_DS(9, d.counts))
    assert mod.evaluate(0, dss, expr, p, be, cs) is None              # other dataset object
    dss[-1] = d
    assert mod.evaluate(0, dss, expr, p, be, cs) == 3.0               # the original again

    # (assigning the identical object is no change: CPython does not report it)
    for field, value in (("dt", float("0.01")), ("dt", 0.02), ("detector_index", 7), ("extra", 1)):
        dss, sess, expr, be, cs = _problem()
        _remember(mod, dss, sess, expr, be, cs)
        assert mod.evaluate(0, dss, expr, p, be, cs) == 3.0
        setattr(dss[1], field, value)                                 # even an equal value
        assert mod.evaluate(0, dss, expr, p, be, cs) is None, field

    dss, sess, expr, be, cs = _problem()
    _remember(mod, dss, sess, expr, be, cs)
    dss[0].counts = dss[0].counts.copy()                              # replaced array
    assert mod.evaluate(0, dss, expr, p, be, cs) is None
    dss, sess, expr, be, cs = _problem()
    _remember(mod, dss, sess, expr, be, cs)
    dss[2].__dict__ = dict(dss[2].__dict__)                           # __dict__ replaced
    assert mod.evaluate(0, dss, expr, p, be, cs) is None


def test_writable_counts_lock_status_and_mlh_errors_miss(fast):
    mod = fast["mod"]
    p = np.ones(3)
    dss, sess, expr, be, cs = _problem()
    _remember(mod, dss, sess, expr, be, cs)
    dss[1].counts.flags.writeable = True          # the only way to edit a frozen array
    assert mod.evaluate(0, dss, expr, p, be, cs) is None
    dss[1].counts.flags.writeable = False
    assert mod.evaluate(0, dss, expr, p, be, cs) == 3.0

    with sess.lock:                               # another thread inside Session.evaluate
        assert mod.evaluate(0, dss, expr, p, be, cs) is None
    calls = fast["calls"]
    fast["rc"] = 5                                # a failing call: the Python path raises
    assert mod.evaluate(0, dss, expr, p, be, cs) is None
    assert fast["calls"] == calls + 1 and not sess.lock.locked()
    fast["rc"] = 0
    fast["bad"] = 17                              # MLH non-positive model: the Python path
    assert mod.evaluate(1, dss, expr, p, be, cs) is None       # raises the reference error
    assert mod.evaluate(0, dss, expr, p, be, cs) == 3.0        # (chi2 has no bad bins)
    fast["bad"] = -1
    assert mod.evaluate(1, dss, expr, p, be, cs) == 1003.0

    mod.forget(object())                          # another session: kept
    assert mod.evaluate(0, dss, expr, p, be, cs) == 3.0
    mod.forget(sess)                              # its session closed: dropped
    assert mod.evaluate(0, dss, expr, p, be, cs) is None and mod.stats()["valid"] == 0


def test_objects_without_dict_are_not_remembered(fast):
    mod = fast["mod"]
    dss = [_Slotted(np.zeros(3))]
    sess = _Sess()
    lock = threading.Lock()
    buf = np.zeros(4)
    ok = mod.remember(sess, dss, object(), None, None, (dss[0].counts,), 1, 1, 1,
                      buf.ctypes.data, buf.ctypes.data, buf.ctypes.data, lock)
    assert ok is False and mod.stats()["valid"] == 0
    assert mod.remember(sess, iter(dss), object(), None, None, (), 1, 1, 1, 0, 0, 0, lock) is False
