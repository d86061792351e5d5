"""C5 (BASELINE.json configs[4]): end-to-end fit with THE REFERENCE'S OWN
minimizer loop -- ``blk.musr.minimize`` from baseline/_ref (musr.py:246-296,
optimize.py Nelder-Mead) -- on 8 x 2^20 bins of the reference's
``generate_synthetic`` data, wall time with the GPU objective plugged in via
``install(blk.musr, blk.theory)`` (the registry musr.py:235 that minimize reads
at call time, musr.py:261-263) vs the reference's stock CPU objective
(``Backend(1)``; ``Backend(cpu_count)`` is probed and the faster one used).

Also reported: this package's ``minimize`` (same iterates, Nelder-Mead run
natively around the device objective).

    python tools/fit_c5.py [cpu_budget_s]     # 0 = run the whole CPU fit
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
import numpy as np

import blk.backend
import blk.musr
import blk.theory
import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import workloads as W

cpu_budget = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0
w = W.c5()
expr = blk.theory.parse(w.expr.source)
bindings = [blk.theory.TheoryBinding(map=tuple(b.map), function_values=tuple(b.function_values))
            for b in w.bindings]
truth = blk.musr.ParameterSet(values=w.params.copy(), names=[f"p{i}" for i in range(6)],
                              step_sizes=np.ones(6))
dss = blk.musr.generate_synthetic(truth=truth, expr=expr, bindings=bindings, n0_slots=w.n0_slots,
                                  nbkg_slots=w.nbkg_slots, nbins=w.nbins, dt=w.dt, seed=w.seed)
start = blk.musr.ParameterSet(values=np.array([0.3, 0.15, 5.0, 0.045, 1000.0, 10.0]),
                              names=["A0", "sigma", "phi_offset", "B", "N0", "Nbkg"],
                              step_sizes=np.array([0.01, 0.01, 1.0, 0.001, 1.0, 0.5]),
                              bounds=[None, (1e-6, np.inf), None, (1e-6, np.inf), None, None],
                              fixed=np.array([False, False, False, False, True, True]))
cpu_backend = blk.backend.Backend(worker_count=1)
out = {"workload": "C5 (8 x 2^20 bins, Eq. 6, chi2; reference generate_synthetic, seed 5)",
       "minimizer": "blk.musr.minimize (baseline/_ref, unmodified)"}

# -- GPU objective through the reference's registry ---------------------------------------
prev = pkg.install(blk.musr, blk.theory)
try:
    blk.musr.OBJECTIVES["chi2"](dss, expr, w.params, cpu_backend)   # session build outside
    t0 = time.perf_counter()
    gpu = blk.musr.minimize("chi2", dss, expr, start, cpu_backend)
    t_gpu = time.perf_counter() - t0
finally:
    pkg.uninstall(blk.musr, prev)
out.update(gpu_fit_s=t_gpu, gpu_evals=gpu.objective_evaluations, gpu_iterations=gpu.iterations,
           gpu_converged=bool(gpu.converged), gpu_chi2=gpu.objective_value,
           gpu_params=gpu.best_parameters.values.tolist(),
           gpu_us_per_eval_incl_nm=1e6 * t_gpu / gpu.objective_evaluations)

# -- this package's minimize (native Nelder-Mead around the device objective) -----------
pstart = pkg.ParameterSet(values=start.values.copy(), names=list(start.names),
                          step_sizes=start.step_sizes.copy(), bounds=list(start.bounds),
                          fixed=start.fixed.copy())
pkg.chi2(dss, expr, w.params)          # session build outside (as for the reference's loop)
t0 = time.perf_counter()
own = pkg.minimize("chi2", dss, expr, pstart)
out.update(pkg_minimize_fit_s=time.perf_counter() - t0,
           pkg_minimize_evals=own.objective_evaluations,
           pkg_minimize_bitwise_equal=bool(np.array_equal(own.best_parameters.values,
                                                          gpu.best_parameters.values)
                                           and own.objective_value == gpu.objective_value))

# -- the reference CPU objective, same loop -------------------------------------------
probe = {}
for k in sorted({1, os.cpu_count() or 1}):
    b = blk.backend.Backend(worker_count=k)
    blk.musr.chi2(dss, expr, w.params, b)
    t0 = time.perf_counter()
    blk.musr.chi2(dss, expr, w.params, b)
    probe[k] = time.perf_counter() - t0
best_k = min(probe, key=probe.get)
cpu_b = blk.backend.Backend(worker_count=best_k)
calls = {"n": 0}
stock = blk.musr.OBJECTIVES["chi2"]


def timed_chi2(*a, **kw):
    calls["n"] += 1
    if cpu_budget and time.perf_counter() - t1 > cpu_budget:
        raise TimeoutError
    return stock(*a, **kw)


blk.musr.OBJECTIVES["chi2"] = timed_chi2
t1 = time.perf_counter()
try:
    cpu = blk.musr.minimize("chi2", dss, expr, start, cpu_b)
    t_cpu = time.perf_counter() - t1
    out.update(cpu_fit_s=t_cpu, cpu_evals=cpu.objective_evaluations, cpu_chi2=cpu.objective_value,
               cpu_params=cpu.best_parameters.values.tolist(),
               params_bitwise_equal=bool(np.array_equal(cpu.best_parameters.values,
                                                        gpu.best_parameters.values)),
               max_rel_param_diff=float(np.max(np.abs(gpu.best_parameters.values - cpu.best_parameters.values)
                                               / np.maximum(np.abs(cpu.best_parameters.values), 1e-300))),
               speedup=t_cpu / t_gpu)
except TimeoutError:
    t_cpu = time.perf_counter() - t1
    per = t_cpu / calls["n"]
    out.update(cpu_fit_s_extrapolated=per * gpu.objective_evaluations, cpu_s_per_eval=per,
               cpu_evals_timed=calls["n"], speedup_extrapolated=per * gpu.objective_evaluations / t_gpu)
finally:
    blk.musr.OBJECTIVES["chi2"] = stock
out.update(cpu_worker_count=best_k, cpu_probe_s={str(k): v for k, v in probe.items()},
           cpu_count=os.cpu_count())
print(json.dumps(out))
