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
