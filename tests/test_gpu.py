"""GPU parity tests: libmusr_b200.so against the reference (golden vectors)
and the CPU oracle, through the drop-in API (musr.chi2 / musr.mlh).

Tolerance (north star): objective values and per-dataset contributions
within 1e-12 relative.  The kernel reproduces the reference's op order and
pairwise tree exactly, so observed differences are transcendental ulps
(~1e-16); exact-value cases are asserted exactly.
"""

import os

import numpy as np
import pytest

import paper_1604_02334_b200 as pkg
from conftest import build_case, hexf, load_golden, rel
from oracle import musr_oracle as O
from paper_1604_02334_b200 import objective, workloads

pytestmark = pytest.mark.gpu
TOL = 1e-14   # "errors within 1e-9" needs <~1e-14 objective agreement
META, ARR = load_golden()


@pytest.fixture(autouse=True)
def _device(gpu_ok):
    yield
    objective.clear_cache()


def _gpu(kind, dss, expr, p, tau=pkg.TAU_MU_US, backend=None):
    fn = pkg.chi2 if kind == "chi2" else pkg.mlh
    total = fn(dss, expr, p, backend, pkg.PhysicsConstants(tau_mu=tau))
    sess = objective.session_for(dss, expr, tau, len(p), backend or pkg.DeviceBackend())
    return total, sess.per_dataset()


def _oracle(kind, dss, expr, p, tau=pkg.TAU_MU_US):
    per = []
    fn = O.chi2 if kind == "chi2" else O.mlh
    return fn(dss, expr, p, tau, musr_error=pkg.MusrError, eval_error=pkg.EvalError,
              per_dataset=per), per


# -- golden vectors from the reference ---------------------------------------------

@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
def test_golden(case):
    dss, expr, p, tau = build_case(case, ARR, pkg)
    for kind, want in case["results"].items():
        if "error" in want:
            with pytest.raises(Exception) as exc:
                _gpu(kind, dss, expr, p, tau)
            assert type(exc.value).__name__ == want["error"]
            assert str(exc.value) == want["message"]
            continue
        total, per = _gpu(kind, dss, expr, p, tau)
        if case["name"].startswith("exact") or (case["name"].startswith("bitwise")
                                                 and kind == "chi2"):
            # exact values, and transcendental-free chi2 (every per-bin op
            # correctly rounded): bit for bit, which pins the reduction tree
            assert total == hexf(want["value"]), (kind, total.hex(), want["value"])
            assert [v.hex() for v in per] == [hexf(v).hex() for v in want["per_dataset"]]
        assert rel(total, hexf(want["value"])) <= TOL, (kind, total, want["value"])
        for a, b in zip(per, want["per_dataset"]):
            assert rel(a, hexf(b)) <= TOL


# -- named workloads vs the oracle ----------------------------------------------------

@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", dict(nbins=1 << 20)),
                                     ("C3", dict(n_hist=16, nbins=1 << 20)),
                                     ("C4", dict(n_hist=8, nbins=1 << 18))])
def test_workloads_vs_oracle(name, kw):
    w = workloads.WORKLOADS[name](**kw)
    dss = workloads.synthesize(w)
    rng = np.random.default_rng(hash(name) % 1000)
    for trial in range(2):
        p = w.params * (1.0 + (0.0 if trial == 0 else 0.03) * rng.standard_normal(len(w.params)))
        for kind in ("chi2", "mlh"):
            g, gp = _gpu(kind, dss, w.expr, p)
            o, op = _oracle(kind, dss, w.expr, p)
            assert rel(g, o) <= TOL, (name, kind, g, o)
            assert max(rel(a, b) for a, b in zip(gp, op)) <= TOL


def test_ragged_fit_ranges_t0_and_tiny_datasets():
    rng = np.random.default_rng(4)
    expr = pkg.parse(workloads.EQ6)
    dss = []
    for j, n in enumerate([1, 2, 255, 256, 257, 2047, 2048, 2049, 5000, 70001, 3, 130000]):
        t0 = int(rng.integers(0, 3)) if n > 10 else 0
        ds = pkg.MusrDataset(j, rng.poisson(200.0, n), 10.0 / 5000, t0,
                             pkg.TheoryBinding(map=(0, 1, 2, 3, 0), function_values=(22.5 * j,)), 4, 5)
        if j % 3 == 1 and n > 10:
            ds.fit_range = (0.5 * ds.dt * n / 10, 0.9 * ds.dt * n)
        dss.append(ds)
    p = np.array([0.25, 0.2, 3.0, 0.05, 200.0, 5.0])
    for kind in ("chi2", "mlh"):
        g, gp = _gpu(kind, dss, expr, p)
        o, op = _oracle(kind, dss, expr, p)
        assert rel(g, o) <= TOL and max(rel(a, b) for a, b in zip(gp, op)) <= TOL


def test_many_datasets_unstaged_path():
    """> 64 datasets: per-dataset rows are read from global memory."""
    w = workloads.c4(n_hist=100, nbins=3000)
    dss = workloads.synthesize(w)
    for kind in ("chi2", "mlh"):
        g, gp = _gpu(kind, dss, w.expr, w.params)
        o, op = _oracle(kind, dss, w.expr, w.params)
        assert rel(g, o) <= TOL and max(rel(a, b) for a, b in zip(gp, op)) <= TOL


def test_non_integer_counts_use_f64_format_and_match():
    rng = np.random.default_rng(5)
    expr = pkg.parse("p[m[0]] * se(t, p[m[1]]) * tf(t, p[m[2]], p[m[3]])")
    dss = [pkg.MusrDataset(0, np.zeros(3), 0.001, 0, pkg.TheoryBinding(map=(0, 1, 2, 3)), 4, 5)]
    dss[0].counts = rng.uniform(0, 5000, 300000)     # non-integer: f64 streams
    p = np.array([0.25, 0.5, 30.0, 1.5, 1000.0, 10.0])
    for kind in ("chi2", "mlh"):
        assert rel(_gpu(kind, dss, expr, p)[0], _oracle(kind, dss, expr, p)[0]) <= TOL


def test_formats_bitwise_identical(monkeypatch):
    w = workloads.c2(n_hist=3, nbins=100000)
    dss = workloads.synthesize(w)
    got = {}
    for fmt in ("auto", "f64"):
        monkeypatch.setenv("MUSR_FORMAT", fmt)
        objective.clear_cache()
        got[fmt] = [_gpu(k, dss, w.expr, w.params)[0] for k in ("chi2", "mlh")]
    assert got["auto"] == got["f64"]


# -- reference-test ports (test_musr.py, test_acceptance.py) ---------------------------

def _flat(counts, dt=0.01, t0=0, j=0):
    return pkg.MusrDataset(j, np.asarray(counts), dt, t0, pkg.TheoryBinding(map=()), 0, 1)


def test_exact_values():
    zero = pkg.parse("0 * t")
    p = np.array([100.0, 5.0])
    ds = _flat(np.zeros(50))
    ds.counts = O.model_expected(ds, zero, p)             # numpy model, as test_musr.py:100-104
    assert pkg.chi2([ds], zero, p) == 0.0
    assert pkg.chi2([_flat([4])], zero, np.array([0.0, 2.0])) == 1.0
    assert pkg.mlh([_flat(np.full(100, 7))], zero, np.array([0.0, 7.0])) == 0.0
    assert pkg.mlh([_flat([0])], zero, np.array([0.0, 3.0])) == 6.0
    base = np.full(200, 9)
    assert pkg.mlh([_flat(base)], pkg.parse("0"), np.array([0.0, 9.0])) == 0.0
    for b in (0, 57, 199):
        for delta in (-1, 1):
            c = base.copy()
            c[b] += delta
            assert pkg.mlh([_flat(c)], pkg.parse("0"), np.array([0.0, 9.0])) > 0.0


def test_mlh_first_nonpositive_bin_in_large_dataset():
    expr = pkg.parse("p[m[0]] * t")
    ds = pkg.MusrDataset(3, np.full(500000, 50), 0.001, 11, pkg.TheoryBinding(map=(2,)), 0, 1)
    # model = (1 * env) * (1 + a*t) + 0 turns non-positive where a*t <= -1
    p = np.array([1.0, 0.0, -1.0 / 300.0])
    with pytest.raises(pkg.MusrError) as exc:
        pkg.mlh([ds], expr, p)
    with pytest.raises(Exception) as ref_exc:
        O.mlh([ds], expr, p, musr_error=pkg.MusrError)
    assert str(exc.value) == str(ref_exc.value)


def test_determinism_and_dataset_split():
    w = workloads.c2(n_hist=4, nbins=200000)
    dss = workloads.synthesize(w)
    a = pkg.chi2(dss, w.expr, w.params)
    assert all(pkg.chi2(dss, w.expr, w.params) == a for _ in range(5))
    folded = 0.0
    for ds in dss:
        folded = folded + pkg.chi2([ds], w.expr, w.params)   # musr.py:190-201
    assert folded == a


def test_collective_path_world1_matches():
    """The NCCL (sharded) handle with world size 1 gives identical bits."""
    w = workloads.c2(n_hist=3, nbins=50000)
    dss = workloads.synthesize(w)
    plain = [pkg.chi2(dss, w.expr, w.params), pkg.mlh(dss, w.expr, w.params)]
    be = pkg.DeviceBackend(collective=True, nccl_id=objective.new_nccl_id())
    coll = [pkg.chi2(dss, w.expr, w.params, be), pkg.mlh(dss, w.expr, w.params, be)]
    assert plain == coll


def test_session_invalidation_on_mutation():
    w = workloads.c1(nbins=4096)
    dss = workloads.synthesize(w)
    a = pkg.chi2(dss, w.expr, w.params)
    dss[0].fit_range = (1.0, 5.0)
    b = pkg.chi2(dss, w.expr, w.params)
    assert b != a and rel(b, O.chi2(dss, w.expr, w.params)) <= TOL
    dss[0].counts = dss[0].counts + 1.0
    assert rel(pkg.chi2(dss, w.expr, w.params), O.chi2(dss, w.expr, w.params)) <= TOL


def test_tile_shape_api_validates():
    """musr_set_tile_shape: only {4, 8, 16} terms x {4, 8, 16} warps, and only
    before the theory and data (the layout and the compiled kernel depend on it)."""
    import ctypes as C

    from paper_1604_02334_b200 import _lib

    lib = _lib.load()
    assert lib.musr_set_tile_shape(None, 8, 8) != 0
    h = C.c_void_p()
    assert lib.musr_open(0, C.byref(h)) == 0
    try:
        for pt, cw in ((8, 32), (3, 8), (8, 2), (32, 8)):
            assert lib.musr_set_tile_shape(h, pt, cw) != 0, (pt, cw)
        assert lib.musr_set_tile_shape(h, 8, 4) == 0
        from paper_1604_02334_b200 import codegen

        frag = codegen.lower(workloads.c1(nbins=4096).expr.ast).source
        log = C.create_string_buffer(1 << 16)
        assert lib.musr_set_theory(h, frag.encode(), log, len(log)) == 0
        assert lib.musr_set_tile_shape(h, 8, 8) != 0          # after the theory: refused
        assert b"before the theory" in lib.musr_last_error(h)
    finally:
        lib.musr_close(h)


def test_small_problem_tile_shape_gives_identical_bits(monkeypatch):
    """A few-tile problem runs with 1024- / 2048-term tiles (8 terms x 4 / 8
    warps, objective.small_problem_tile_shape); its chi2 / MLH values -- transcendental
    theory, per dataset and total -- equal the default 4096-term shape's bit for
    bit, so a rank's shape choice can never change a sharded result."""
    for w in (workloads.c1(nbins=1 << 16), workloads.c2(n_hist=3, nbins=70001)):
        dss = workloads.synthesize(w)
        got = {}
        for forced in (False, True):
            objective.clear_cache()
            if forced:
                monkeypatch.setenv("MUSR_CWARPS", "16")          # the default shape
            for kind in ("chi2", "mlh"):
                total, per = _gpu(kind, dss, w.expr, w.params)
                sess = objective.session_for(dss, w.expr, pkg.TAU_MU_US, len(w.params),
                                             pkg.DeviceBackend())
                assert sess.tile_shape == (None if forced else
                                           ((8, 4) if len(dss) == 1 else (8, 8)))
                got[(forced, kind)] = (total, list(per))
            monkeypatch.delenv("MUSR_CWARPS", raising=False)
        for kind in ("chi2", "mlh"):
            assert got[(False, kind)] == got[(True, kind)], kind
            assert rel(got[(False, kind)][0], _oracle(kind, dss, w.expr, w.params)[0]) <= TOL


def test_concurrent_calls_from_threads_are_serialised():
    """Several threads calling the drop-in objective on one cached problem (the
    C fast path and, when its lock is busy, the Python path) get exactly the
    values of sequential calls: evaluations on a handle never interleave."""
    import threading

    w = workloads.c2(n_hist=4, nbins=40000)
    dss = workloads.synthesize(w)
    rng = np.random.default_rng(21)
    P = [w.params * (1.0 + 0.02 * rng.standard_normal(len(w.params))) for _ in range(24)]
    want = [(pkg.chi2(dss, w.expr, p), pkg.mlh(dss, w.expr, p)) for p in P]
    got = {}
    errors = []

    def worker(k):
        try:
            for rep in range(5):
                for i in range(k, len(P), 4):
                    got[(k, rep, i)] = (pkg.chi2(dss, w.expr, P[i]), pkg.mlh(dss, w.expr, P[i]))
        except BaseException as exc:        # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert len(got) == 5 * len(P)
    for (k, rep, i), v in got.items():
        assert v == want[i], (k, rep, i)


def test_fast_path_repeated_calls_and_every_invalidation():
    """The C fast path (csrc/musr_pyfast.c) answers repeated calls; every edit
    the reference would see on its next call (musr.py:181-232 reads the
    datasets each time) gives the oracle's new value, bit for bit where the
    slow path does."""
    from paper_1604_02334_b200 import _lib

    w = workloads.c2(n_hist=3, nbins=5000)
    dss = workloads.synthesize(w)
    p = np.array(w.params, dtype=np.float64)
    cs = pkg.PhysicsConstants()
    first = pkg.chi2(dss, w.expr, p, None, cs)          # slow path, remembered
    assert _lib.pyfast().stats()["valid"] == 1
    for _ in range(3):
        assert pkg.chi2(dss, w.expr, p, None, cs) == first
    assert rel(first, O.chi2(dss, w.expr, p)) <= TOL
    q = p.copy()
    q[0] *= 1.001                                       # new parameters: fast path, new value
    assert pkg.chi2(dss, w.expr, q, None, cs) == O.chi2(dss, w.expr, q) or \
        rel(pkg.chi2(dss, w.expr, q, None, cs), O.chi2(dss, w.expr, q)) <= TOL
    assert pkg.mlh(dss, w.expr, q, None, cs) == pkg.mlh(dss, w.expr, q.tolist(), None, cs)

    def check():
        g = pkg.chi2(dss, w.expr, p, None, cs)
        assert rel(g, O.chi2(dss, w.expr, p)) <= TOL
        assert pkg.chi2(dss, w.expr, p, None, cs) == g  # and again through the fast path
        return g

    dss[1].fit_range = (0.5, 3.0)
    a = check()
    dss[0].dt = dss[0].dt * 1.5
    b = check()
    dss.pop()
    c = check()
    assert len({first, a, b, c}) == 4
    dss[0].counts.flags.writeable = True                # the one way to edit in place
    dss[0].counts[100] += 7.0
    check()
    dss[0].counts.flags.writeable = True                # (frozen again by the rebuild)
    dss[0].counts[200] += 3.0
    check()

    # an MLH model that goes non-positive after a remembered call raises as the reference
    m = pkg.parse("p[m[0]] * t")
    ds = [pkg.MusrDataset(detector_index=4, counts=np.full(64, 5.0), dt=0.1, t0_bin=3,
                          binding=pkg.TheoryBinding(map=(0,)), n0_slot=1, nbkg_slot=2)]
    good = np.array([0.5, 10.0, 1.0])
    v = pkg.mlh(ds, m, good, None, cs)
    assert pkg.mlh(ds, m, good, None, cs) == v
    bad = np.array([-5.0, 10.0, 1.0])
    with pytest.raises(pkg.MusrError) as e_gpu:
        pkg.mlh(ds, m, bad, None, cs)
    with pytest.raises(Exception) as e_ref:
        O.mlh(ds, m, bad)
    assert str(e_gpu.value) == str(e_ref.value)


# -- fits through the reference minimizer loop -----------------------------------------

def _eq6_problem(n_det, nbins, seed, dt):
    expr = pkg.parse(workloads.EQ6)
    truth = np.array([0.25, 0.2, 0.0, 0.05, 1000.0, 10.0])
    bindings = [pkg.TheoryBinding(map=(0, 1, 2, 3, 0), function_values=(float(ph),))
                for ph in pkg.default_phases(n_det)]
    dss = O.generate_synthetic(
        lambda j, c, d, t0, b, n0, nb: pkg.MusrDataset(j, c, d, t0, b, n0, nb),
        truth, expr, bindings, [4] * n_det, [5] * n_det, nbins, dt, seed)
    start = pkg.ParameterSet(values=np.array([0.3, 0.15, 5.0, 0.045, 1000.0, 10.0]),
                             names=["A0", "sigma", "phi_offset", "B", "N0", "Nbkg"],
                             step_sizes=np.array([0.01, 0.01, 1.0, 0.001, 1.0, 0.5]),
                             bounds=[None, (1e-6, np.inf), None, (1e-6, np.inf), None, None],
                             fixed=np.array([False, False, False, False, True, True]))
    return dss, expr, start


def test_fit_parameters_match_cpu_objective():
    """Same minimizer loop, GPU objective vs CPU oracle objective: fitted
    parameters within 1e-9 relative (north-star fit parity)."""
    dss, expr, start = _eq6_problem(4, 20000, 7, 0.0005)
    gpu = pkg.minimize("chi2", dss, expr, start)
    cpu = pkg.minimize("chi2", dss, expr, start, objective_fn=lambda p: O.chi2(dss, expr, p))
    free = ~start.fixed
    g, c = gpu.best_parameters.values[free], cpu.best_parameters.values[free]
    assert np.all(np.abs(g - c) <= 1e-9 * np.abs(c) + 1e-15), (g, c)
    assert rel(gpu.objective_value, cpu.objective_value) <= TOL
    assert gpu.objective_value == pkg.chi2(dss, expr, gpu.best_parameters.values)


def test_acceptance_criterion_1_fit_recovery():
    """test_acceptance.py:115-167 on the GPU objective: 16 x 50000 bins."""
    dss, expr, start = _eq6_problem(16, 50000, 31, 0.0001953125)
    res = pkg.minimize("chi2", dss, expr, start)
    best = res.best_parameters
    ndf = pkg.degrees_of_freedom(dss, best)
    assert 0.9 <= res.objective_value / ndf <= 1.1
    slot = best.slot("B")

    def chi2_of_b(b):
        p = best.values.copy()
        p[slot] = b
        return pkg.chi2(dss, expr, p)

    def crossing(direction):
        step, lo = 1e-5, best.values[slot]
        while chi2_of_b(lo + direction * step) < res.objective_value + 1.0:
            step *= 2.0
        a, c = lo, lo + direction * step
        for _ in range(60):
            mid = 0.5 * (a + c)
            if chi2_of_b(mid) < res.objective_value + 1.0:
                a = mid
            else:
                c = mid
        return 0.5 * (a + c)

    se = 0.5 * (crossing(+1.0) - crossing(-1.0))
    assert abs(best.values[slot] - 0.05) <= 3.0 * se


# -- batched evaluation -----------------------------------------

@pytest.mark.parametrize("name,kw", [("C1", dict(nbins=1 << 14)), ("C2", dict(n_hist=5, nbins=100000)),
                                     ("C3", dict(n_hist=3, nbins=70001))])
def test_batch_bitwise_equals_single(name, kw):
    """Every row of chi2_batch / mlh_batch equals the scalar call bit for bit,
    across chunk boundaries (MUSR_KMAX = 8 points per launch)."""
    w = workloads.WORKLOADS[name](**kw)
    dss = workloads.synthesize(w)
    rng = np.random.default_rng(11)
    for n_points in (1, 3, 8, 13):
        P = w.params * (1.0 + 0.02 * rng.standard_normal((n_points, len(w.params))))
        for kind, one, many in (("chi2", pkg.chi2, pkg.chi2_batch), ("mlh", pkg.mlh, pkg.mlh_batch)):
            got = many(dss, w.expr, P)
            want = np.array([one(dss, w.expr, p) for p in P])
            assert got.shape == (n_points,)
            assert np.array_equal(got.view(np.int64), want.view(np.int64)), (name, kind, n_points)
    assert pkg.chi2_batch(dss, w.expr, np.zeros((0, len(w.params)))).shape == (0,)


def test_batch_many_datasets_and_collective_path():
    w = workloads.c4(n_hist=70, nbins=2000)            # > 64 datasets: unstaged metadata
    dss = workloads.synthesize(w)
    P = np.repeat(w.params[None, :], 9, axis=0)
    P[:, 1] *= np.linspace(0.9, 1.1, 9)
    want = np.array([pkg.chi2(dss, w.expr, p) for p in P])
    assert np.array_equal(pkg.chi2_batch(dss, w.expr, P), want)
    be = pkg.DeviceBackend(collective=True, nccl_id=objective.new_nccl_id())
    assert np.array_equal(pkg.chi2_batch(dss, w.expr, P, be), want)


def test_batch_mlh_error_is_first_failing_point():
    expr = pkg.parse("p[m[0]] * t")
    ds = pkg.MusrDataset(3, np.full(50000, 50), 0.001, 11, pkg.TheoryBinding(map=(2,)), 0, 1)
    good = np.array([1.0, 0.0, 0.0])
    bad1 = np.array([1.0, 0.0, -1.0 / 30.0])
    bad2 = np.array([1.0, 0.0, -1.0 / 20.0])
    with pytest.raises(pkg.MusrError) as exc:
        pkg.mlh_batch([ds], expr, np.array([good, bad2, bad1]))
    with pytest.raises(pkg.MusrError) as one:
        pkg.mlh([ds], expr, bad2)
    assert str(exc.value) == str(one.value)
    assert pkg.mlh_batch([ds], expr, np.array([good, good]))[1] == pkg.mlh([ds], expr, good)


def test_minimize_batched_simplex_identical_to_unbatched():
    """minimize() batches the initial simplex and shrink points; the fit is
    bit-identical to the one-call-per-point loop."""
    dss, expr, start = _eq6_problem(4, 20000, 7, 0.0005)
    batched = pkg.minimize("chi2", dss, expr, start)
    single = pkg.minimize("chi2", dss, expr, start,
                          objective_fn=lambda p: pkg.chi2(dss, expr, p))
    assert np.array_equal(batched.best_parameters.values, single.best_parameters.values)
    assert batched.objective_value == single.objective_value
    assert batched.objective_evaluations == single.objective_evaluations


# -- full BASELINE sizes and pipeline-depth invariance -----------------------------------

def test_full_size_c4_sampled_parity():
    """C4 at its full size (64 x 2^22 bins, one GPU): per-dataset values of a
    sample of datasets against the oracle (each dataset's sum is independent of
    the others), and the total equals the left fold of the per-dataset values."""
    w = workloads.c4()
    dss = workloads.synthesize(w)
    for kind in ("chi2", "mlh"):
        total, per = _gpu(kind, dss, w.expr, w.params)
        folded = 0.0
        for v in per:
            folded = folded + v                                  # musr.py:190-201
        assert folded == total
        for j in (0, 21, 42, 63):
            o, _ = _oracle(kind, [dss[j]], w.expr, w.params)
            assert rel(per[j], o) <= TOL, (kind, j, per[j], o)


@pytest.mark.parametrize("src", ["p[m[0]] * sg(t, p[m[1]]) * tf(t, p[m[2]] + f[m[0]], 135.538809 * p[m[3]])",
                                 "p[m[0]] * t + (p[m[1]] - p[m[3]]) / (2.5 * p[m[2]] + 1)",
                                 "p[m[0]] * exp(-p[m[1]] * t) * cos(p[m[3]] ^ 1.5 * t) + log(p[m[2]]) * 0.01"])
def test_host_uniform_rows_match_device_prologue(monkeypatch, src):
    """The per-call host rows (musr_set_uniform_program: the parameter-only values,
    rotation tables, N0, Nbkg passed inline) against the CTA prologue's device rows
    (MUSR_DEVICE_ROWS): bit-identical objectives for arithmetic-only uniform parts,
    within 1e-15 where exp / log / cos / sin / pow of parameters enter (host libm vs
    device library), and both within 1e-14 of the oracle."""
    expr = pkg.parse(src)
    rng = np.random.default_rng(len(src))
    dss = []
    for j in range(5):
        n = [4095, 70001, 1, 9000, 130001][j]
        dt = 10.0 / max(n, 64)
        lam = 900.0 * np.exp(-np.arange(n) * dt / 2.197019) + 10.0
        dss.append(pkg.MusrDataset(j, rng.poisson(lam), dt, j % 3 if n > 8 else 0, pkg.TheoryBinding(
            map=(0, 1, 2, 3), function_values=(30.0 * j,)), 4, 5))
    p = np.array([0.2, 0.3, 4.0, 0.05, 1000.0, 10.0])
    got = {}
    for mode in ("host", "device"):
        if mode == "device":
            monkeypatch.setenv("MUSR_DEVICE_ROWS", "1")
        objective.clear_cache()
        got[mode] = [_gpu(k, dss, expr, p) for k in ("chi2", "mlh")]
    arith = "exp" not in src
    for i, kind in enumerate(("chi2", "mlh")):
        (h, hp), (d, dp) = got["host"][i], got["device"][i]
        if arith:
            assert h == d and list(hp) == list(dp), kind
        else:
            assert rel(h, d) <= 1e-15 and max(rel(a, b) for a, b in zip(hp, dp)) <= 1e-14, kind
        assert rel(h, _oracle(kind, dss, expr, p)[0]) <= TOL


def test_host_uniform_rows_values():
    """musr_eval_uniform_rows for the C2 theory: U = (A0, sigma, 2 pi k B, (phi + f) pi / 180)
    exactly as numpy float64 scalars give them, rotation entries D_j = W (j dt) exactly
    with cos / sin within an ulp of numpy's, then N0, Nbkg."""
    import ctypes as C
    w = workloads.c2(n_hist=3, nbins=4096)
    dss = workloads.synthesize(w)
    p = w.params
    pkg.chi2(dss, w.expr, p)
    sess = objective.session_for(dss, w.expr, pkg.TAU_MU_US, len(p), pkg.DeviceBackend())
    pt = sess.tile_shape[0] if sess.tile_shape else 8          # rotation entries per thread run
    row = sess.lowered.n_uniform_reg + 4 * pt * sess.lowered.n_rotations + 2
    rows = np.zeros((3, row))
    pc = np.ascontiguousarray(p, dtype=np.float64)
    assert sess._lib.musr_eval_uniform_rows(sess._handle, pc.ctypes.data, len(pc), rows.ctypes.data) == 0
    f64 = np.float64
    for j, ds in enumerate(dss):
        m, fv = ds.binding.map, ds.binding.function_values
        W = f64(2.0 * np.pi) * (f64(workloads.K_MHZ_PER_T) * f64(p[m[3]]))
        assert rows[j, 0] == p[m[0]] and rows[j, 1] == p[m[1]] and rows[j, 2] == W
        assert rows[j, 3] == ((f64(p[m[2]]) + f64(fv[m[4]])) * f64(np.pi)) / f64(180.0)
        for k in range(1, pt):
            D = W * (f64(k) * f64(ds.dt))
            e = rows[j, 4 + 4 * k: 8 + 4 * k]
            assert e[0] == D and abs(e[1] - np.cos(D)) <= 2.3e-16 and abs(e[2] - np.sin(D)) <= 2.3e-16
        assert rows[j, -2] == p[ds.n0_slot] and rows[j, -1] == p[ds.nbkg_slot]


def test_pipeline_depth_and_large_table_invariance(monkeypatch):
    """The TMA pipeline depth is picked at run time (the deepest that fits next
    to the count table and the staged rows): 1, 2 and 3 stages give identical
    bits, also with a 4096-entry count table and 64 staged datasets."""
    rng = np.random.default_rng(9)
    w = workloads.c4(n_hist=64, nbins=20000)
    dss = workloads.synthesize(w)
    dss[5].counts[7] = 4095.0                      # table_size 4096 (64 KB of shared memory)
    p = w.params.copy()
    p[4] = 1500.0 + 200.0 * rng.standard_normal()
    got = {}
    for st in ("1", "2", "3"):
        monkeypatch.setenv("MUSR_STAGES", st)
        objective.clear_cache()
        got[st] = [_gpu(k, dss, w.expr, p)[0] for k in ("chi2", "mlh")]
    assert got["1"] == got["2"] == got["3"]
    for i, kind in enumerate(("chi2", "mlh")):
        assert rel(got["3"][i], _oracle(kind, dss, w.expr, p)[0]) <= TOL


# -- multi-rank: shared host results (two ranks on this GPU) -----------------------------

def _shared_rank(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be = pkg.DeviceBackend(device=0, rank=rank, world=world,
                           shared_results=objective.shared_result_buffer(dist))
    w = workloads.c2(n_hist=7, nbins=1 << 16)          # 7 datasets: uneven shards
    dss = workloads.synthesize(w)
    rng = np.random.default_rng(3)
    res = []
    for _ in range(4):
        p = w.params * (1.0 + 0.03 * rng.standard_normal(len(w.params)))
        res.append([pkg.chi2(dss, w.expr, p, be), pkg.mlh(dss, w.expr, p, be)])
    res.append(list(pkg.chi2_batch(dss, w.expr, np.array([w.params, 1.01 * w.params]), be)))
    expr = pkg.parse("p[m[0]] * t")                     # MLH error raised on every rank
    bad = [pkg.MusrDataset(j, np.full(400000 - 1000 * j, 50), 0.001, 11, pkg.TheoryBinding(map=(2,)), 0, 1)
           for j in range(3)]
    try:
        pkg.mlh(bad, expr, np.array([1.0, 0.0, -1.0 / 300.0]), be)
        res.append("no error")
    except pkg.MusrError as exc:
        res.append(str(exc))
    import pickle

    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump([[float(v) for v in x] if not isinstance(x, str) else x for x in res], f)
    objective.clear_cache()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_shared_host_results_two_ranks_match_one_gpu(tmp_path, world):
    """Two (four) ranks -- processes -- on this GPU, each owning a contiguous
    share of the datasets, combine their results through the shared host
    buffer: every rank gets the one-GPU values bit for bit, batched calls and
    the MLH error included.  (No rank's kernel waits on another's: only the
    hosts poll the buffer, so sharing one GPU cannot deadlock.)"""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_shared_rank, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    w = workloads.c2(n_hist=7, nbins=1 << 16)
    dss = workloads.synthesize(w)
    rng = np.random.default_rng(3)
    want = []
    for _ in range(4):
        p = w.params * (1.0 + 0.03 * rng.standard_normal(len(w.params)))
        want.append([pkg.chi2(dss, w.expr, p), pkg.mlh(dss, w.expr, p)])
    want.append(list(pkg.chi2_batch(dss, w.expr, np.array([w.params, 1.01 * w.params]))))
    expr = pkg.parse("p[m[0]] * t")
    bad = [pkg.MusrDataset(j, np.full(400000 - 1000 * j, 50), 0.001, 11, pkg.TheoryBinding(map=(2,)), 0, 1)
           for j in range(3)]
    with pytest.raises(pkg.MusrError) as exc:
        pkg.mlh(bad, expr, np.array([1.0, 0.0, -1.0 / 300.0]))
    want.append(str(exc.value))
    import pickle

    want = [[float(v) for v in x] if not isinstance(x, str) else x for x in want]
    for r in range(world):
        with open(tmp_path / f"rank{r}.pkl", "rb") as f:
            assert pickle.load(f) == want, r


def test_long_parameter_vector_not_inline():
    """n_p > 64 (here 3 + 3 x 24 = 75): p goes through the device buffer, not the
    kernel parameters; values and batched values still match the oracle."""
    w = workloads.c2(n_hist=24, nbins=30000)
    dss = workloads.synthesize(w)
    assert len(w.params) > 64
    rng = np.random.default_rng(8)
    P = np.array([w.params * (1.0 + 0.02 * rng.standard_normal(len(w.params))) for _ in range(3)])
    for kind in ("chi2", "mlh"):
        for p in P:
            g, gp = _gpu(kind, dss, w.expr, p)
            o, op = _oracle(kind, dss, w.expr, p)
            assert rel(g, o) <= TOL and max(rel(a, b) for a, b in zip(gp, op)) <= TOL
        fnb = pkg.chi2_batch if kind == "chi2" else pkg.mlh_batch
        fn = pkg.chi2 if kind == "chi2" else pkg.mlh
        assert list(fnb(dss, w.expr, P)) == [fn(dss, w.expr, p) for p in P]


def test_native_minimize_identical_to_python_loop():
    """pkg.minimize runs the Nelder-Mead loop natively (musr_minimize); the
    Python loop over the same GPU objective gives the same fit bit for bit, and
    an objective error raised mid-fit surfaces with the reference's message."""
    w = workloads.c5(n_hist=4, nbins=1 << 16)
    dss = workloads.synthesize(w)
    start = pkg.ParameterSet(values=np.array([0.3, 0.15, 5.0, 0.045, 1000.0, 10.0]),
                             names=["A0", "sigma", "phi", "B", "N0", "Nbkg"],
                             step_sizes=np.array([0.01, 0.01, 1.0, 0.001, 1.0, 0.5]),
                             bounds=[None, (1e-6, np.inf), None, (1e-6, np.inf), None, None],
                             fixed=np.array([False, False, False, False, True, True]))
    for kind, fn in (("chi2", pkg.chi2), ("mlh", pkg.mlh)):
        native = pkg.minimize(kind, dss, w.expr, start)
        loop = pkg.minimize(kind, dss, w.expr, start, objective_fn=lambda q: fn(dss, w.expr, q))
        assert np.array_equal(native.best_parameters.values, loop.best_parameters.values), kind
        assert native.objective_value == loop.objective_value
        assert (native.iterations, native.objective_evaluations, native.converged) == \
               (loop.iterations, loop.objective_evaluations, loop.converged)
    # MLH turns non-positive mid-fit: the data fall faster than the envelope, the
    # first reflection takes a below -1 / t_max and the model below zero
    expr = pkg.parse("p[m[0]] * t")
    t = np.arange(400000) * 0.001
    counts = np.round(np.maximum(0.0, 50.0 * np.exp(-t / pkg.TAU_MU_US) * (1.0 - 0.003 * t)))
    ds = pkg.MusrDataset(0, counts, 0.001, 0, pkg.TheoryBinding(map=(0,)), 1, 2)
    bad = pkg.ParameterSet(values=np.array([0.0, 50.0, 0.0]), names=["a", "N0", "Nbkg"],
                           step_sizes=np.array([0.01, 1.0, 1.0]),
                           fixed=np.array([False, True, True]))
    with pytest.raises(pkg.MusrError) as a:
        pkg.minimize("mlh", [ds], expr, bad)
    with pytest.raises(pkg.MusrError) as b:
        pkg.minimize("mlh", [ds], expr, bad, objective_fn=lambda q: pkg.mlh([ds], expr, q))
    assert str(a.value) == str(b.value)
