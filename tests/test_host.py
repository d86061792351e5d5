"""Host-side logic that needs no GPU: the C ABI surface, the device math
library compiled for the host, error resolution, sharding, the restated
Nelder-Mead driver, and the multi-rank result combination (gloo)."""

import ctypes as C
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import _lib, objective
from paper_1604_02334_b200.codegen import lower
from paper_1604_02334_b200.optimize import MinimizeConfig, nelder_mead

ROOT = Path(__file__).resolve().parents[1]


# -- C ABI ------------------------------------------------------------------------

def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "musr_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|void|const char\*)\s+(musr_\w+)\s*\(", header, re.M))
    assert len(declared) >= 14
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    typed = {name for name, _, _ in _lib.SIGNATURES}
    assert declared == typed, declared ^ typed


def test_library_reports_no_device_cleanly():
    lib = _lib.load()
    n = C.c_int(-1)
    assert lib.musr_device_count(C.byref(n)) == 0
    if n.value == 0:
        h = C.c_void_p()
        assert lib.musr_open(0, C.byref(h)) != 0
        assert b"device" in lib.musr_global_error().lower()
    assert lib.musr_set_tile_shape(None, 8, 8) != 0      # NULL handle: an error, no crash


def test_no_cpu_fallback_without_device():
    """Objective calls raise loudly when no device is present."""
    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    ds = pkg.MusrDataset(0, np.arange(10), 0.1, 0, pkg.TheoryBinding(map=()), 0, 1)
    with pytest.raises(_lib.MusrDeviceError):
        pkg.chi2([ds], pkg.parse("0 * t"), np.array([1.0, 2.0]))


# -- device math (host build of csrc/musr_math.cuh, IEEE fma from libm) ------------

@pytest.fixture(scope="module")
def mathlib(tmp_path_factory):
    out = tmp_path_factory.mktemp("math") / "libmath_host.so"
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-Wno-unknown-pragmas",
                    "-shared", "-fPIC", "-o", str(out),
                    str(ROOT / "tools" / "mathgen" / "math_host.cpp"), "-lm"], check=True)
    lib = C.CDLL(str(out))

    def call(name, *arrs):
        res = np.empty_like(arrs[0])
        args = [a.ctypes.data_as(C.c_void_p) for a in arrs]
        getattr(lib, name)(*args, res.ctypes.data_as(C.c_void_p), C.c_long(len(res)))
        return res

    return call


def test_device_exp_within_one_ulp(mathlib):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-708, 708, 400000), rng.uniform(-50, 1, 400000),
                        [0.0, -0.0, 708.0, -708.0, 709.0, -745.0, np.inf, -np.inf, np.nan]])
    y = mathlib("v_exp", x)
    with np.errstate(over="ignore"):
        ref = np.exp(x)
    ulps = np.abs(y.view(np.int64) - ref.view(np.int64))
    finite = np.isfinite(ref) & (ref > 1e-300)
    assert ulps[finite].max() <= 1
    assert np.array_equal(np.isnan(y), np.isnan(ref))


def test_device_cos_sin_absolute_error(mathlib):
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-1e4, 1e4, 300000), rng.uniform(-2**20, 2**20, 100000),
                        np.arange(-500, 500) * np.pi / 2, [0.0, 2.0**20, -2.0**21, 1e300]])
    for name, f in (("v_cos", np.cos), ("v_sin", np.sin)):
        y = mathlib(name, x)
        assert np.abs(y - f(x)).max() <= 4e-16, name


def test_anchored_exp_within_two_ulp(mathlib):
    """musr_exp_anchored (runs of consecutive bins, |x - x0| < 2^-10) against numpy exp."""
    rng = np.random.default_rng(5)
    n = 400_000
    x0 = np.concatenate([rng.uniform(-700, 700, n), rng.uniform(-20, 0, n)])
    x = x0 + rng.uniform(-2.0**-10, 2.0**-10, 2 * n) * rng.choice([1.0, 1e-3, 1e-6], 2 * n)
    y = mathlib("v_exp_anchored", x, x0)
    ref = np.exp(x)
    keep = ~np.isnan(y)
    assert keep.mean() > 0.99
    assert np.abs(y[keep].view(np.int64) - ref[keep].view(np.int64)).max() <= 2
    far = mathlib("v_exp_anchored", np.array([1.0 + 2.0**-9, 0.0]), np.array([1.0, 2.0**-9]))
    assert np.isnan(far).all()  # outside the window: the kernel recomputes exactly


def test_scaled_anchored_exp_bitwise(mathlib):
    """exp(c * y) anchored on y with c^k-scaled coefficients (codegen's form for
    the -0.5 of sg / stg) is bit-identical to the anchored exp of x = c * y,
    including the window test."""
    rng = np.random.default_rng(8)
    n = 300_000
    c = rng.choice([-0.5, 0.5, -2.0, 4.0, -0.25, -1.0], n)
    y0 = rng.uniform(-300, 300, n) / np.abs(c)
    y = y0 + rng.uniform(-2.0**-9, 2.0**-9, n) * rng.choice([1.0, 1e-2, 1e-6], n) / np.abs(c)
    got = mathlib("v_exp_anchored_k", y, y0, c)
    want = mathlib("v_exp_anchored", c * y, c * y0)
    assert np.isnan(got).sum() == np.isnan(want).sum() > 0
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_log_exponent_table_bitwise(mathlib):
    """musr_log_fast_k (exponent folded into a 1024-entry table, the MLH hot
    path) equals musr_log_fast bit for bit on [0.043, 22) and hands everything
    else (k outside [-4, 4), zero, negative, subnormal, inf, NaN) to the exact path."""
    rng = np.random.default_rng(9)
    x = np.concatenate([np.exp(rng.uniform(np.log(0.6875 / 16), np.log(1.375 * 8), 400_000)),
                        1.0 + rng.uniform(-0.05, 0.05, 100_000), [1.0, 0.6875 / 16, 1.375 * 8 * (1 - 2**-52)]])
    got, want = mathlib("v_log_k", x), mathlib("v_log", x)
    assert not np.isnan(got).any()
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    out = np.array([0.6875 / 16 * (1 - 2**-52), 1.375 * 8, 100.0, 1e-3, 0.0, -1.0, 5e-324, np.inf, np.nan])
    assert np.isnan(mathlib("v_log_k", out)).all()


def test_err_rcp_fast_every_integer_count(tmp_path_factory, mathlib):
    """The chi2 kernel's in-kernel error path (branch-free sqrt and reciprocal,
    used for counts beyond its table and for the f64 format) equals IEEE
    max(1, sqrt(k)) and 1/err for every integer k in [1, 2^23)."""
    lib = C.CDLL(str(next(tmp_path_factory.getbasetemp().glob("math*")) / "libmath_host.so"))
    lib.v_err_rcp_scan.restype = C.c_long
    assert lib.v_err_rcp_scan(C.c_long(1), C.c_long(1 << 23)) == 0
    rng = np.random.default_rng(12)
    x = np.concatenate([np.exp(rng.uniform(0.0, 36.0, 500_000)), 1.0 + rng.uniform(0, 1, 100_000)])
    assert np.array_equal(mathlib("v_sqrt_fast", x), np.sqrt(x))
    assert np.isnan(mathlib("v_sqrt_fast", np.array([0.5, 0.0, -4.0, 2.0**53, np.inf, np.nan]))).all()


def test_pow_anchor_within_two_ulp(mathlib):
    """musr_pow_fast (the anchored pow's anchor: exp(b log x) carried in
    extended precision) against libm pow; musr_rcp_approx to 1 ulp."""
    import math
    rng = np.random.default_rng(7)
    n = 200_000
    x = np.exp(rng.uniform(-20, 20, n))
    b = rng.uniform(-4, 4, n)
    keep = np.abs(b * np.log(x)) < 700
    x, b = x[keep], b[keep]
    y = mathlib("v_pow_fast", x, b)
    ref = np.array([math.pow(u, v) for u, v in zip(x, b)])
    assert not np.isnan(y).any()
    assert np.abs(y.view(np.int64) - ref.view(np.int64)).max() <= 2
    bad = mathlib("v_pow_fast", np.array([0.0, -1.0, np.inf, 1e300]), np.array([1.5, 1.5, 1.5, 3.0]))
    assert np.isnan(bad).all()   # outside the fast domain: the kernel recomputes exactly
    r = mathlib("v_rcp_approx", x)
    assert np.abs(r.view(np.int64) - (1.0 / x).view(np.int64)).max() <= 1


def test_rotated_cos_absolute_error(mathlib):
    """The tf rotation: cos(a0 + D + e) from (cos a0, sin a0), (cos D, sin D) and e."""
    rng = np.random.default_rng(6)
    n = 400_000
    a0 = np.round(rng.uniform(-500, 500, n) * 2.0**20) / 2.0**20  # a0 + D exact in fp64
    D = np.round(rng.uniform(0, 0.05, n) * 2.0**40) / 2.0**40
    e = rng.uniform(-1e-13, 1e-13, n)
    y = mathlib("v_cos_rotated", a0, D, e)
    ref = np.cos(a0 + D) - np.sin(a0 + D) * e  # e^2 ~ 1e-26 is far below an ulp
    assert np.abs(y - ref).max() <= 5e-16


def test_markstein_division_is_exact(mathlib):
    rng = np.random.default_rng(2)
    n = 1_000_000
    d = rng.integers(0, 10**6, n).astype(np.float64)
    e = np.maximum(1.0, np.sqrt(d))
    y = 1.0 / e
    for a in (rng.standard_normal(n) * e, d - rng.uniform(0, 2e6, n), np.round(rng.standard_normal(n) * 30),
              rng.standard_normal(n) * 1e300, rng.uniform(-1e-300, 1e-300, n)):
        q = mathlib("v_div_y", a, e, y)
        assert np.array_equal(q.view(np.int64), (a / e).view(np.int64))
    a = np.array([np.inf, -np.inf, np.nan, 0.0, -0.0])
    b = np.array([1.0, 3.0, 2.0, 7.0, 7.0])
    q = mathlib("v_div_y", a, b, 1.0 / b)
    ref = a / b
    assert np.array_equal(q[:2], ref[:2]) and np.isnan(q[2])
    assert np.array_equal(np.signbit(q[3:]), np.signbit(ref[3:]))


def test_device_log_within_one_ulp(mathlib):
    """musr_log_fast (MLH term) against glibc log, which is correctly rounded here."""
    import math
    rng = np.random.default_rng(3)
    n = 200_000
    d = rng.integers(1, 5000, n).astype(np.float64)
    x = np.concatenate([rng.uniform(0.5, 2, n), 1 + rng.uniform(-1e-3, 1e-3, n),
                        np.exp(rng.uniform(-700, 700, n)), d / rng.uniform(1e-3, 5000, n),
                        [1.0, 2.0, 0.5, np.nextafter(1.0, 2.0), np.nextafter(1.0, 0.0)]])
    y = mathlib("v_log", x)
    ref = np.array([math.log(v) for v in x])
    assert np.abs(y.view(np.int64) - ref.view(np.int64)).max() <= 1
    bad = mathlib("v_log", np.array([0.0, -1.0, np.inf, np.nan, 5e-324]))
    assert np.isnan(bad).all()  # outside the fast domain: the kernel recomputes exactly


def test_device_fast_division_is_exact(mathlib):
    """musr_div_fast (MLH quotient d / m) is the IEEE quotient on its domain."""
    rng = np.random.default_rng(4)
    n = 1_000_000
    for a, b in ((rng.integers(1, 5000, n).astype(np.float64), rng.uniform(1e-3, 5000, n)),
                 (np.exp(rng.uniform(-340, 340, n)), np.exp(rng.uniform(-340, 340, n)))):
        q = mathlib("v_div_fast", a, b)
        assert not np.isnan(q).any()
        assert np.array_equal(q.view(np.int64), (a / b).view(np.int64))
    out = mathlib("v_div_fast", np.array([1.0, 0.0, 1e300, 1.0]), np.array([0.0, 1.0, 1.0, -1.0]))
    assert np.isnan(out).all()


# -- error resolution ------------------------------------------------------------

def _ds(j, counts, bmap=(), f=(), n0=0, nbkg=1, t0=0, fit=None):
    ds = pkg.MusrDataset(j, np.asarray(counts), 0.01, t0, pkg.TheoryBinding(map=bmap, function_values=f),
                         n0, nbkg)
    ds.fit_range = fit
    return ds


@pytest.mark.parametrize("src,ds,n_p,want", [
    ("p[m[3]] * t", _ds(0, [5, 6], (0,)), 2, ("EvalError", "slot 3 not covered by map of length 1")),
    ("p[m[0]] + t", _ds(0, [5, 6], (7,)), 2,
     ("EvalError", "map entry m[0]=7 out of range for 'p' array of length 2")),
    ("f[m[1]] + p[m[0]] * t", _ds(0, [5, 6], (0, 2), (0.5,)), 2,
     ("EvalError", "map entry m[1]=2 out of range for 'f' array of length 1")),
    ("t + 1 / (2 - 2)", _ds(0, [5, 6]), 2, ("ZeroDivisionError", "float division by zero")),
    ("0 * t", _ds(0, [5, 6], n0=9), 2, ("IndexError", "index 9 is out of bounds for axis 0 with size 2")),
    ("0 * t", _ds(0, [5, 6], n0=-2, nbkg=-1), 2, None),
])
def test_static_errors(src, ds, n_p, want):
    err = objective._static_error(ds, lower(pkg.parse(src).ast), n_p, pkg.MusrError, pkg.EvalError)
    if want is None:
        assert err is None
    else:
        assert (type(err).__name__, str(err)) == want


def test_empty_fit_range_detected_at_prepare():
    low = lower(pkg.parse("0 * t").ast)
    prep = objective._prepare(1, _ds(1, [1, 2, 3], fit=(100.0, 200.0)), low, 2.197019, 2,
                              pkg.MusrError, pkg.EvalError, need_streams=False)
    assert str(prep.error) == "detector 1: empty fit range"
    prep = objective._prepare(0, _ds(0, np.arange(100), t0=3, fit=(0.1, 0.5)), low, 2.197019, 2,
                              pkg.MusrError, pkg.EvalError, need_streams=True)
    t = (np.arange(100) - 3) * 0.01
    mask = (t >= 0.1) & (t <= 0.5)
    assert prep.first == np.flatnonzero(mask)[0] and prep.n_terms == mask.sum()
    assert np.array_equal(prep.envelope, np.exp(-t / 2.197019)[mask])
    assert np.array_equal(prep.errors, np.maximum(1.0, np.sqrt(np.arange(100.0)))[mask])


# -- sharding ------------------------------------------------------------------

def test_shard_assignment_contiguous_balanced():
    assert objective.shard_assignment([10] * 64, 8) == [r for r in range(8) for _ in range(8)]
    assert objective.shard_assignment([5, 5], 1) == [0, 0]
    rng = np.random.default_rng(3)
    for _ in range(200):
        n = rng.integers(1, 10000, int(rng.integers(1, 70)))
        world = int(rng.integers(1, 9))
        owner = objective.shard_assignment(n, world)
        assert owner == sorted(owner) and max(owner) < world      # contiguous, in range
        loads = np.bincount(owner, weights=n, minlength=world)
        assert loads.max() <= n.sum() / world + n.max()


def _ll_words(value: float, epoch: int):
    """The objective kernel's LL encoding of one fp64 result (musr_kernel.cuh
    musr_ll_put): two 8-byte words (32-bit half << 32) | epoch."""
    b = int(np.float64(value).view(np.uint64))
    return [((b >> 32) << 32) | epoch, ((b & 0xffffffff) << 32) | epoch]


def _gloo_worker(rank, world, port, q):
    """One rank of the shared-results exchange with the product's own host code:
    shard_assignment (which datasets this rank owns), shared_result_buffer (the
    ranks' common mapping) and musr_collect_results (decode + the ordered fold
    musr_eval runs).  Only the device kernel is stood in for: the rank's owned
    datasets are summed by the oracle and written as the kernel's LL words."""
    import ctypes

    import torch.distributed as dist

    from oracle import musr_oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    expr = pkg.parse("p[m[0]] * sg(t, p[m[1]])")
    dss = [_ds(j, rng.poisson(300, int(rng.integers(500, 3000))), (2, 3)) for j in range(7)]
    G = len(dss)
    owner = objective.shard_assignment([len(d.counts) for d in dss], world)
    addr, nbytes = objective.shared_result_buffer(dist, 1 << 16)
    words = (ctypes.c_uint64 * (nbytes // 8)).from_address(addr)
    lib = _lib.load()
    out = []
    for epoch in (5, 6, 7):                     # double-buffered by epoch parity
        p = np.array([1000.0, 10.0, 0.25, 0.3 + 0.01 * epoch])
        base = (epoch & 1) * 4 * G
        for j, ds in enumerate(dss):
            if owner[j] == rank:
                w = _ll_words(O.chi2([ds], expr, p), epoch) + _ll_words(0.0, epoch)
                for k in range(4):
                    words[base + 4 * j + k] = w[k]
        dist.barrier()
        per = np.zeros(G)
        bad = np.zeros(G, dtype=np.int64)
        tot = C.c_double()
        rc = lib.musr_collect_results(
            ctypes.cast(ctypes.addressof(words) + 8 * base, C.POINTER(C.c_uint64)), G, epoch,
            per.ctypes.data_as(C.POINTER(C.c_double)), bad.ctypes.data_as(C.POINTER(C.c_int64)),
            C.byref(tot))
        stale = lib.musr_collect_results(
            ctypes.cast(ctypes.addressof(words) + 8 * base, C.POINTER(C.c_uint64)), G, epoch + 2,
            None, None, None)
        out.append((rc, tot.value, O.chi2(dss, expr, p), bool((bad == -1).all()), stale))
        dist.barrier()
    q.put((rank, out, sorted(set(owner))))
    dist.destroy_process_group()


def test_sharded_combination_is_exact_gloo():
    """Two gloo ranks combine their shards' results through the product's
    shared buffer and fold: every rank's total equals the one-process value
    bit for bit (each slot has exactly one writer; the fold order is fixed)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert res[0][2] == [0, 1]                    # both ranks own datasets
    for rank, out, _ in res:
        for rc, total, single, none_bad, stale in out:
            assert rc == 0 and total == single and none_bad, rank
            assert stale == 7                     # MUSR_ERR_PEER: words of another epoch


def _shm_worker(rank, world, port, q):
    import ctypes

    import torch.distributed as dist

    from paper_1604_02334_b200 import objective

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    addr, nbytes = objective.shared_result_buffer(dist, 1 << 16)
    words = (ctypes.c_uint64 * (nbytes // 8)).from_address(addr)
    zero = all(w == 0 for w in words[:64])               # zero-filled
    dist.barrier()
    words[rank] = 1000 + rank                            # each rank writes its slot
    dist.barrier()
    leftovers = [f for f in os.listdir("/dev/shm") if f.startswith("musr_b200_")]
    q.put((rank, [words[r] for r in range(world)], addr % 64, leftovers, zero))
    dist.destroy_process_group()


def test_shared_result_buffer_is_one_mapping_gloo():
    """The ranks' result buffer (musr_open_shared's host side): one zero-filled
    mapping seen by every rank, aligned, its /dev/shm name already removed."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_shm_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, seen, align, leftovers, zero in res:
        assert zero and seen == [1000, 1001] and align == 0
        assert leftovers == []     # rank 0 unlinked the name once every rank had mapped it


# -- restated Nelder-Mead (optimize.py:41-146) -------------------------------------

def test_minimize_hooks():
    params = pkg.ParameterSet(values=np.array([0.0]), names=["x"], step_sizes=np.array([0.5]))
    res = pkg.minimize("chi2", [], pkg.parse("0 * t"), params,
                       objective_fn=lambda p: (p[0] - 3.0) ** 2)
    assert res.converged and abs(res.best_parameters.values[0] - 3.0) < 1e-6
    with pytest.raises(Exception, match="not finite"):
        pkg.minimize("chi2", [], pkg.parse("0 * t"), params, objective_fn=lambda p: float("nan"))
    fixed = pkg.ParameterSet(values=np.array([0.0, 5.0]), names=["a", "b"],
                             step_sizes=np.ones(2), fixed=np.array([True, True]))
    res = pkg.minimize("chi2", [], pkg.parse("0 * t"), fixed, objective_fn=lambda p: 1.5)
    assert res.iterations == 0 and res.objective_evaluations == 1 and res.objective_value == 1.5


@pytest.mark.ref
def test_nelder_mead_identical_to_reference(ref):
    rosen = lambda x: float(sum(100.0 * (x[1:] - x[:-1] ** 2) ** 2 + (1 - x[:-1]) ** 2))
    bowl = lambda x: float(np.sum((x - np.arange(len(x))) ** 2 * (1 + np.arange(len(x)))))
    cases = [(rosen, [-1.2, 1.0], [0.1, 0.1], None, None),
             (rosen, [0.5, 0.5, 0.5, 0.5], [0.2] * 4, [-2] * 4, [0.9] * 4),
             (bowl, [5.0] * 6, [1.0] * 6, None, None),
             (bowl, [3.0], [0.5], [1.0], [2.0])]
    for fn, x0, st, lo, hi in cases:
        for cfg_args in ({}, {"max_evaluations": 37}, {"restarts": 0, "tol_f": 1e-4}):
            a = nelder_mead(fn, x0, st, lo, hi, MinimizeConfig(**cfg_args))
            b = ref.optimize.nelder_mead(fn, x0, st, lo, hi, ref.optimize.MinimizeConfig(**cfg_args))
            assert np.array_equal(a.x, b.x) and a.fun == b.fun
            assert (a.iterations, a.evaluations, a.converged) == (b.iterations, b.evaluations, b.converged)
            # the batched simplex / shrink path (fn_batch) takes the same decisions
            calls = []

            def fb(X, fn=fn):
                calls.append(len(X))
                return np.array([fn(x) for x in X])

            c = nelder_mead(fn, x0, st, lo, hi, MinimizeConfig(**cfg_args), fb)
            assert np.array_equal(c.x, b.x) and c.fun == b.fun
            assert (c.iterations, c.evaluations, c.converged) == (b.iterations, b.evaluations, b.converged)
            assert len(x0) == 1 or calls


def _native_nm(fn, x0, steps, lo, hi, tol_f=1e-9, budget=0, restarts=1):
    """musr_nm_run (the native loop behind musr_minimize) over a Python objective."""
    lib = _lib.load()
    n = len(x0)
    CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int,
                     C.POINTER(C.c_double))

    def cb(user, xs, k, nn, fs):
        for i in range(k):
            fs[i] = float(fn(np.array(xs[i * nn:(i + 1) * nn])))
        return 0

    keep = CB(cb)
    x0 = np.minimum(np.maximum(np.asarray(x0, float), lo), hi)
    f0 = float(fn(x0))
    d = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    best, fail = np.zeros(n), np.zeros(n)
    bf, it, ev, conv = C.c_double(), C.c_int64(), C.c_int64(), C.c_int()
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    a = [d(x0), d(steps), d(lo), d(hi)]
    rc = lib.musr_nm_run(n, P(a[0]), f0, P(a[1]), P(a[2]), P(a[3]), tol_f, budget or 400 * n,
                         restarts, C.cast(keep, C.c_void_p), None, P(best), C.byref(bf),
                         C.byref(it), C.byref(ev), C.byref(conv), P(fail))
    assert rc == 0
    return best, bf.value, it.value, ev.value, bool(conv.value)


@pytest.mark.parametrize("speculate", ["0", "1"])
@pytest.mark.parametrize("case", ["rosen2", "rosen5_bounded", "bowl_budget", "nan_region", "one_d"])
def test_native_nelder_mead_bitwise_equal_to_python(case, speculate, monkeypatch):
    """The native loop (musr_minimize's core) reproduces optimize.nelder_mead
    bit for bit: iterates, values, iteration and evaluation counts -- also when
    it evaluates each iteration's reflection, expansion and contraction points
    as one speculative batch (MUSR_NM_SPECULATE=1, what musr_minimize does for
    small problems)."""
    monkeypatch.setenv("MUSR_NM_SPECULATE", speculate)
    from paper_1604_02334_b200.optimize import MinimizeConfig, nelder_mead

    rosen = lambda x: float(np.sum(100.0 * (x[1:] - x[:-1] ** 2) ** 2 + (1 - x[:-1]) ** 2))
    cfgs = {
        "rosen2": (rosen, [-1.2, 1.0], [0.1, 0.1], [-np.inf] * 2, [np.inf] * 2, 0),
        "rosen5_bounded": (rosen, [0.5, 0.2, -0.3, 1.5, 0.9], [0.2] * 5, [-1.0, 0.1, -2, 0.5, 0.0],
                           [1.5, 3.0, 2.0, 1.2, 2.0], 0),
        "bowl_budget": (lambda x: float(np.dot(x - 3.0, x - 3.0)), [0.0, 10.0, -4.0], [1.0, 0.5, 2.0],
                        [-np.inf] * 3, [np.inf] * 3, 37),
        "nan_region": (lambda x: float("nan") if x[0] > 1.7 else float((x[0] - 2) ** 2 + x[1] ** 2),
                       [0.0, 1.0], [0.6, 0.3], [-np.inf] * 2, [np.inf] * 2, 0),
        "one_d": (lambda x: float(np.cos(x[0]) + 0.1 * x[0] ** 2), [2.0], [0.3], [-5.0], [5.0], 0),
    }
    fn, x0, steps, lo, hi, budget = cfgs[case]
    lo, hi = np.asarray(lo, float), np.asarray(hi, float)
    ref = nelder_mead(fn, x0, steps, lo, hi, MinimizeConfig(max_evaluations=budget))
    best, bf, it, ev, conv = _native_nm(fn, x0, steps, lo, hi, budget=budget)
    assert np.array_equal(best.view(np.int64), ref.x.view(np.int64)), (best, ref.x)
    assert (bf == ref.fun) or (np.isnan(bf) and np.isnan(ref.fun))
    assert (it, ev, conv) == (ref.iterations, ref.evaluations, ref.converged)


def test_native_nelder_mead_reports_failing_point():
    """A nonzero status from the objective aborts the native loop with that
    status and the failing point in fail_x (musr_minimize re-raises there)."""
    lib = _lib.load()
    CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int,
                     C.POINTER(C.c_double))
    seen = []

    def cb(user, xs, k, n, fs):
        for i in range(k):
            x = [xs[i * n + j] for j in range(n)]
            seen.append(x)
            if len(seen) == 5:
                return 100
            fs[i] = (x[0] - 1.0) ** 2 + (x[1] + 2.0) ** 2
        return 0

    keep = CB(cb)
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    x0, st = np.array([0.0, 0.0]), np.array([0.5, 0.5])
    lo, hi = np.full(2, -np.inf), np.full(2, np.inf)
    best, fail = np.zeros(2), np.zeros(2)
    rc = lib.musr_nm_run(2, P(x0), 5.0, P(st), P(lo), P(hi), 1e-9, 800, 1,
                         C.cast(keep, C.c_void_p), None, P(best), None, None, None, None, P(fail))
    assert rc == 100
    assert fail.tolist() == seen[4]


def test_speculative_nelder_mead_fails_where_the_sequential_loop_fails(monkeypatch):
    """An objective that fails on a region of parameter space: the speculative
    loop (batched reflection / expansion / contractions) must abort at exactly
    the point the sequential loop aborts at -- a speculative point it would
    never have evaluated must not fail the fit -- or finish identically."""
    lib = _lib.load()
    CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int,
                     C.POINTER(C.c_double))

    def cb(user, xs, k, n, fs):
        for i in range(k):
            x = [xs[i * n + j] for j in range(n)]
            if x[0] > 1.6 and x[1] < -0.9:             # the "raising" region
                return 100
            fs[i] = (x[0] - 1.0) ** 2 + 3.0 * (x[1] + 0.5) ** 2 + 0.1 * x[0] * x[1]
        return 0

    keep = CB(cb)
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    lo, hi = np.full(2, -np.inf), np.full(2, np.inf)
    outcomes = {}
    for start in ([0.0, 0.0], [2.0, 1.0], [-1.0, -2.0], [1.3, 0.3], [2.5, -0.5], [1.5, -0.6]):
        for spec in ("0", "1"):
            monkeypatch.setenv("MUSR_NM_SPECULATE", spec)
            x0, st = np.array(start), np.array([0.5, 0.5])
            best, fail = np.zeros(2), np.full(2, np.nan)
            bf, it, ev = C.c_double(), C.c_int64(), C.c_int64()
            f0 = (start[0] - 1.0) ** 2 + 3.0 * (start[1] + 0.5) ** 2 + 0.1 * start[0] * start[1]
            rc = lib.musr_nm_run(2, P(x0), f0, P(st), P(lo), P(hi), 1e-12, 800, 1,
                                 C.cast(keep, C.c_void_p), None, P(best), C.byref(bf),
                                 C.byref(it), C.byref(ev), None, P(fail))
            outcomes[(tuple(start), spec)] = (rc, fail.tobytes() if rc else best.tobytes(),
                                              None if rc else (bf.value, it.value, ev.value))
        assert outcomes[(tuple(start), "0")] == outcomes[(tuple(start), "1")], start
    assert any(v[0] == 100 for v in outcomes.values())     # the region is reached somewhere
    assert any(v[0] == 0 for v in outcomes.values())


# -- session cache (objective.session_for) with a stand-in for the device session ----

class _StubSession:
    built = 0

    def __init__(self, datasets, expr, tau_mu, n_p, backend):
        type(self).built += 1
        self.n = len(datasets)
        self._handle = object()
        self._frozen = []

    def close(self):
        objective._FROZEN.release(self)
        self._handle = None


@pytest.fixture
def stub_sessions(monkeypatch):
    objective.clear_cache()
    monkeypatch.setattr(objective, "Session", _StubSession)
    _StubSession.built = 0
    yield _StubSession
    objective.clear_cache()


def test_session_cache_sees_list_edits_and_unhashable_ranges(stub_sessions):
    expr = pkg.parse("p[m[0]] * t")
    dss = [_ds(j, np.arange(10.0) + j, (2,)) for j in range(3)]
    be = objective.DeviceBackend()
    s1 = objective.session_for(dss, expr, 2.197019, 3, be)
    assert objective.session_for(dss, expr, 2.197019, 3, be) is s1 and stub_sessions.built == 1
    dss.pop()                                             # same list object, edited in place
    s2 = objective.session_for(dss, expr, 2.197019, 3, be)
    assert s2 is not s1 and s2.n == 2
    dss.append(dss[0])                                    # re-appending an existing dataset
    assert objective.session_for(dss, expr, 2.197019, 3, be).n == 3
    dss[1].fit_range = [0.1, 0.5]                         # list (the reference accepts any pair)
    objective.session_for(dss, expr, 2.197019, 3, be)
    dss[1].fit_range = np.array([0.1, 0.6])
    objective.session_for(dss, expr, 2.197019, 3, be)


def test_session_cache_freezes_counts_and_rebuilds_after_unfreeze(stub_sessions):
    """The reference reads ds.counts on every call (musr.py:196): an in-place
    edit of a cached array must never be answered from the stale device copy.
    It raises at the write site; after an explicit unfreeze the next call
    rebuilds from the current contents; flags are restored on eviction."""
    expr = pkg.parse("p[m[0]] * t")
    ds = _ds(0, np.arange(10.0), (2,))
    be = objective.DeviceBackend()
    s1 = objective.session_for([ds], expr, 2.197019, 3, be)
    with pytest.raises(ValueError):
        ds.counts[3] += 1.0
    same = [ds]
    assert objective.session_for(same, expr, 2.197019, 3, be) is s1
    ds.counts.flags.writeable = True
    ds.counts[3] += 1.0
    s2 = objective.session_for(same, expr, 2.197019, 3, be)
    assert s2 is not s1 and stub_sessions.built == 2 and not ds.counts.flags.writeable
    objective.clear_cache()
    assert ds.counts.flags.writeable
    shared = np.arange(5.0)                               # one array under two sessions
    a, b = _ds(0, shared, (2,)), _ds(1, shared, (2,))
    a.counts = shared
    b.counts = shared
    objective.session_for([a], expr, 2.197019, 3, be)
    objective.session_for([b], expr, 2.197019, 4, be)
    assert not shared.flags.writeable


def test_small_problem_tile_shape(monkeypatch):
    """Few-tile problems take 1024- or 2048-term tiles of 8 terms x 4 / 8 warps
    (musr_set_tile_shape); everything else keeps the default; explicit
    MUSR_PT / MUSR_CWARPS win.  The terms per thread never change, so values
    are bit-identical for every shape (the GPU suite checks it)."""
    monkeypatch.delenv("MUSR_PT", raising=False)
    monkeypatch.delenv("MUSR_CWARPS", raising=False)
    assert objective.small_problem_tile_shape([1 << 16]) == (8, 4)          # C1: 16 tiles
    assert objective.small_problem_tile_shape([(1 << 16) + 1]) == (8, 8)    # 17 tiles
    assert objective.small_problem_tile_shape([4097] * 32) == (8, 8)        # 2 tiles each
    assert objective.small_problem_tile_shape([1 << 18]) == (8, 8)          # 64 tiles
    assert objective.small_problem_tile_shape([(1 << 18) + 1]) is None      # 65 tiles
    assert objective.small_problem_tile_shape([1 << 20] * 8) is None        # C2
    assert objective.small_problem_tile_shape([]) is None                   # rank without data
    monkeypatch.setenv("MUSR_PT", "8")
    assert objective.small_problem_tile_shape([1 << 16]) is None
