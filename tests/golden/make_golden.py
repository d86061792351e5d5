"""Generate golden vectors for the objective path from the REFERENCE package.

Run in the build container (the reference is importable there, not on GPU
hosts):

    python tests/golden/make_golden.py          # writes tests/golden/musr_golden.{json,npz}

Every case is evaluated by the reference's own ``blk.musr.chi2`` / ``mlh``
(pkg/src/blk/musr.py:181-232) with ``Backend(1)``; errors are recorded as
(type name, message).  Inputs mirror the reference's tests:

* ``crit2_*``   acceptance criterion 2 problems (test_acceptance.py:170-225)
* ``theory_*``  the C1/C2/C3 benchmark theories at small
                sizes with t0 > 0 and explicit fit ranges
* ``dsl_*``     per-bin ``log``, per-bin-exponent ``pow`` / ``^``, ``exp(t)``,
                uniform-exponent squares (theory.py:91-98, 450-452)
* ``bitwise_*`` transcendental-free theories over ragged lengths (1, 2, 4095,
                4096, 4097, 65539) with t0 > 0 and fit ranges: every per-bin op is
                correctly rounded, so GPU chi2 must equal them bit for bit
* ``exact_*``   exact-value tests (test_musr.py:99-180, test_acceptance.py:228-255)
* ``err_*``     error semantics (empty range, map errors, non-positive MLH,
                literal division by zero, N0 slot out of bounds)
* ``pairwise``  pairwise_sum of ragged lengths (backend.py:79-95)
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def main() -> None:
    sys.path.insert(0, str(REF))
    from blk import musr  # noqa: E402  (reference)
    from blk.backend import Backend, pairwise_sum  # noqa: E402
    from blk.theory import TheoryBinding, parse  # noqa: E402

    backend = Backend(1)
    cases = []
    arrays = {}

    def dataset(j, counts, dt, t0, bmap, fvals, n0, nbkg, fit_range=None, raw=False):
        ds = musr.MusrDataset(detector_index=j, counts=np.asarray(counts), dt=dt, t0_bin=t0,
                              binding=TheoryBinding(map=tuple(bmap), function_values=tuple(fvals)),
                              n0_slot=n0, nbkg_slot=nbkg)
        if raw:  # the reference tests assign non-integer counts directly
            ds.counts = np.asarray(counts, dtype=np.float64)
        ds.fit_range = fit_range
        return ds

    def record(name, source, dss, p, kinds=("chi2", "mlh"), tau=None):
        constants = musr.PhysicsConstants() if tau is None else musr.PhysicsConstants(tau_mu=tau)
        expr = parse(source)
        meta = {"name": name, "expr": source, "p": [float(x).hex() for x in p],
                "tau_mu": float(constants.tau_mu).hex(), "datasets": [], "results": {}}
        for j, ds in enumerate(dss):
            key = f"{name}/{j}"
            arrays[key] = np.asarray(ds.counts, dtype=np.float64)
            meta["datasets"].append({
                "counts": key, "detector_index": ds.detector_index, "dt": float(ds.dt).hex(),
                "t0_bin": int(ds.t0_bin), "map": list(ds.binding.map),
                "f": [float(v).hex() for v in ds.binding.function_values],
                "n0_slot": int(ds.n0_slot), "nbkg_slot": int(ds.nbkg_slot),
                "fit_range": None if ds.fit_range is None else [float(ds.fit_range[0]).hex(),
                                                                float(ds.fit_range[1]).hex()],
            })
        for kind in kinds:
            fn = musr.chi2 if kind == "chi2" else musr.mlh
            try:
                total = fn(dss, expr, np.asarray(p, dtype=np.float64), backend, constants)
                per = [fn([ds], expr, np.asarray(p, dtype=np.float64), backend, constants)
                       for ds in dss]
                meta["results"][kind] = {"value": float(total).hex(),
                                         "per_dataset": [float(v).hex() for v in per]}
            except Exception as exc:  # noqa: BLE001 - recorded as the expected error
                meta["results"][kind] = {"error": type(exc).__name__, "message": str(exc)}
        cases.append(meta)

    rng = np.random.default_rng(20260417)

    # -- acceptance criterion 2 style ---------------------------------------------
    crng = np.random.default_rng(41)
    for case in range(10):
        dss = [dataset(k, crng.integers(1, 400, int(crng.integers(100, 2000))), 0.01,
                       int(crng.integers(0, 4)), (2, 3), (), 0, 1)
               for k in range(int(crng.integers(1, 4)))]
        p = [crng.uniform(50, 300), crng.uniform(0, 20), crng.uniform(0.05, 0.4),
             crng.uniform(0.05, 2.0)]
        record(f"crit2_{case}", "p[m[0]] * se(t, p[m[1]])", dss, p)

    # -- benchmark theories, small, ragged, t0 > 0, fit ranges -----------------------
    K = musr.GAMMA_MU / (2.0 * np.pi)
    eq6 = f"p[m[0]] * sg(t, p[m[1]]) * tf(t, p[m[2]] + f[m[4]], {K!r} * p[m[3]])"
    theories = [
        ("C1", "p[m[0]] * se(t, p[m[1]]) * tf(t, p[m[2]], p[m[3]])",
         [0.25, 0.5, 30.0, 1.5, 1000.0, 10.0], lambda j: ((0, 1, 2, 3), ()), 4, 5),
        ("C2", eq6, [0.25, 0.2, 0.0, 0.05, 1000.0, 10.0],
         lambda j: ((0, 1, 2, 3, 0), (45.0 * j,)), 4, 5),
        ("C3", "p[m[0]] * stg(t, p[m[1]]) * se(t, p[m[2]]) + p[m[3]] * ge(t, p[m[4]], p[m[5]])",
         [0.2, 0.3, 0.1, 0.05, 0.5, 1.5, 1000.0, 10.0], lambda j: ((0, 1, 2, 3, 4, 5), ()), 6, 7),
    ]
    for name, src, p, bind, n0, nbkg in theories:
        expr = parse(src)
        truth = musr.ParameterSet(values=np.array(p), names=[f"x{i}" for i in range(len(p))],
                                  step_sizes=np.ones(len(p)))
        for variant, (nbins, t0, rng_fit) in enumerate(
                [(5000, 0, None), (4099, 7, (0.5, 8.0)), (2049, 0, (0.0, 9.99))]):
            bindings = [TheoryBinding(map=bind(j)[0], function_values=bind(j)[1]) for j in range(3)]
            dss = musr.generate_synthetic(truth, expr, bindings, [n0] * 3, [nbkg] * 3,
                                          nbins=nbins, dt=10.0 / nbins, seed=100 + variant)
            for ds in dss:  # t0 shift after synthesis (ge() is NaN for t < 0)
                ds.t0_bin = t0
                ds.fit_range = rng_fit
            pert = np.array(p) * (1.0 + 0.02 * rng.standard_normal(len(p)))
            record(f"theory_{name}_{variant}", src, dss, pert)

    # -- DSL builtins on a per-bin argument: log, per-bin-exponent pow, exp(t) ---------
    dsl = [
        ("log", "p[m[0]] * log(1 + p[m[1]] * t)", [0.05, 0.7]),
        ("pow_bin_exp", "p[m[0]] * pow(1 + t / 10, -p[m[1]] * t)", [0.3, 0.2]),
        ("caret_bin_exp", "p[m[0]] * (t / 10) ^ (0.5 * t)", [0.2, 0.0]),
        ("exp_t", "p[m[0]] * exp(t) / 10000 + p[m[1]] * log(2 + t)", [0.5, 0.02]),
        ("sq_uniform", "p[m[0]] * sin(3 * t) ^ 2 + p[m[1]] * sqrt(t)", [0.2, 0.05]),
    ]
    for name, src, a in dsl:
        expr = parse(src)
        pv = np.array(a + [1000.0, 10.0])
        truth = musr.ParameterSet(values=pv, names=[f"x{i}" for i in range(len(pv))],
                                  step_sizes=np.ones(len(pv)))
        bindings = [TheoryBinding(map=(0, 1)) for _ in range(2)]
        dss = musr.generate_synthetic(truth, expr, bindings, [2] * 2, [3] * 2, nbins=6007,
                                      dt=10.0 / 6007, seed=300)
        dss[1].t0_bin = 5
        dss[1].fit_range = (0.25, 9.0)
        record(f"dsl_{name}", src, dss, pv * (1.0 + 0.01 * rng.standard_normal(len(pv))))

    # -- transcendental-free theories (every per-bin op correctly rounded): the GPU
    #    total must equal these bit for bit, which pins the reduction tree -----------
    for name, src, a in [("affine", "p[m[0]] * t + p[m[1]]", [0.01, -0.02]),
                         ("rational", "p[m[0]] / (1 + t)", [0.3, 0.0]),
                         ("zero", "0", [0.0, 0.0])]:
        pv = np.array(a + [1000.0, 10.0])
        dss = []
        for j, (n, t0, fr) in enumerate([(1, 0, None), (2, 0, None), (4095, 3, None),
                                         (4096, 0, (0.001, 9.0)), (4097, 11, None),
                                         (65539, 0, (0.5, 7.5))]):
            cnt = np.random.default_rng(500 + j).poisson(900.0 * np.exp(-np.arange(n) / n) + 10)
            dss.append(dataset(j, cnt, 10.0 / max(n, 100), t0, (0, 1), (), 2, 3, fit_range=fr))
        record(f"bitwise_{name}", src, dss, pv, kinds=("chi2", "mlh"))

    # -- exact-value tests --------------------------------------------------------
    zero = "0 * t"
    p = np.array([100.0, 5.0])
    ds = dataset(0, np.zeros(50), 0.01, 0, (), (), 0, 1)
    ds.counts = musr.model_expected(ds, parse(zero), p)
    record("exact_perfect_chi2", zero, [ds], p, kinds=("chi2",))
    record("exact_single_bin", zero, [dataset(0, [4], 0.01, 0, (), (), 0, 1)], [0.0, 2.0])
    record("exact_mlh_floor", "0", [dataset(0, np.full(200, 9), 0.01, 0, (), (), 0, 1)],
           [0.0, 9.0])
    record("exact_mlh_zero_bin", zero, [dataset(0, [0], 0.01, 0, (), (), 0, 1)], [0.0, 3.0])
    record("exact_mlh_integer", zero, [dataset(0, np.full(100, 7), 0.01, 0, (), (), 0, 1)],
           [0.0, 7.0])

    # -- error semantics ------------------------------------------------------------
    record("err_empty_range", zero,
           [dataset(0, [1, 2, 3], 0.01, 0, (), (), 0, 1),
            dataset(1, [1, 2, 3], 0.01, 0, (), (), 0, 1, fit_range=(100.0, 200.0))], [1.0, 0.0])
    record("err_slot_not_covered", "p[m[3]] * t", [dataset(0, [5, 6], 0.01, 0, (0,), (), 0, 1)],
           [1.0, 1.0])
    record("err_map_p_range", "p[m[0]] + t", [dataset(0, [5, 6], 0.01, 0, (7,), (), 0, 1)],
           [1.0, 1.0])
    record("err_map_f_range", "f[m[1]] + p[m[0]] * t",
           [dataset(0, [5, 6], 0.01, 0, (0, 2), (0.5,), 0, 1)], [1.0, 1.0])
    record("err_mlh_nonpositive", zero,
           [dataset(0, [3, 3], 0.01, 0, (), (), 0, 1), dataset(1, [1, 2, 3], 0.01, 2, (), (), 2, 3)],
           [1.0, 2.0, 0.0, 0.0])
    record("err_mlh_then_empty", zero,
           [dataset(0, [3, 3], 0.01, 0, (), (), 2, 3),
            dataset(1, [1, 2, 3], 0.01, 0, (), (), 0, 1, fit_range=(50.0, 60.0))],
           [1.0, 2.0, 0.0, 0.0])
    record("err_zero_division", "t + 1 / (2 - 2)", [dataset(0, [5, 6], 0.01, 0, (), (), 0, 1)],
           [1.0, 1.0])
    record("err_n0_slot", zero, [dataset(0, [5, 6], 0.01, 0, (), (), 9, 1)], [1.0, 1.0])
    record("ok_negative_slot", zero, [dataset(0, [5, 6, 7], 0.01, 0, (), (), -2, -1)],
           [1.0, 2.0, 3.0])
    record("ok_nan_model_propagates", "p[m[0]] * t", [dataset(0, [5, 6, 7], 0.01, 0, (2,), (), 0, 1)],
           [10.0, 1.0, float("nan")])

    # -- pairwise tree ---------------------------------------------------------------
    lengths = [0, 1, 2, 3, 7, 64, 255, 256, 257, 1000, 2047, 2048, 2049, 100003]
    sums = {}
    for n in lengths:
        x = rng.uniform(-1e3, 1e3, n)
        arrays[f"pairwise/{n}"] = x
        sums[str(n)] = float(pairwise_sum(x)).hex()

    meta = {"generator": "tests/golden/make_golden.py", "numpy": np.__version__,
            "reference": "pkg/src/blk (Backend(1))", "cases": cases,
            "pairwise": {"lengths": lengths, "sums": sums}}
    (OUT / "musr_golden.json").write_text(json.dumps(meta, indent=1))
    np.savez_compressed(OUT / "musr_golden.npz", **{k.replace("/", "__"): v for k, v in arrays.items()})
    print(f"wrote {len(cases)} cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()
