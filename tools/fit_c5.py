"""C5: end-to-end fit with the reference minimizer loop (restated Nelder-Mead,
bitwise identical to pkg/src/blk/optimize.py), GPU objective vs the CPU oracle
objective on the same 8 x 2^20-bin data (BASELINE.json configs[4])."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1604_02334_b200 as pkg
from paper_1604_02334_b200 import workloads as W
from oracle import musr_oracle as O

cpu_budget = float(sys.argv[1]) if len(sys.argv) > 1 else 0.0   # seconds; 0 = full CPU fit
w = W.c5()
dss = W.synthesize(w)
start = pkg.ParameterSet(values=np.array([0.3, 0.15, 5.0, 0.045, 1000.0, 10.0]),
                         names=["A0", "sigma", "phi_offset", "B", "N0", "Nbkg"],
                         step_sizes=np.array([0.01, 0.01, 1.0, 0.001, 1.0, 0.5]),
                         bounds=[None, (1e-6, np.inf), None, (1e-6, np.inf), None, None],
                         fixed=np.array([False, False, False, False, True, True]))
pkg.chi2(dss, w.expr, w.params)                       # session build (upload + JIT) outside
t0 = time.perf_counter()
gpu = pkg.minimize("chi2", dss, w.expr, start)
t_gpu = time.perf_counter() - t0
out = {"workload": "C5 (8 x 2^20 bins, Eq. 6, chi2)", "gpu_fit_s": t_gpu,
       "gpu_evals": gpu.objective_evaluations, "gpu_iterations": gpu.iterations,
       "gpu_converged": bool(gpu.converged), "gpu_chi2": gpu.objective_value,
       "gpu_params": gpu.best_parameters.values.tolist(),
       "gpu_us_per_eval_incl_nm": 1e6 * t_gpu / gpu.objective_evaluations}
calls = {"n": 0}


def cpu_obj(p):
    calls["n"] += 1
    if cpu_budget and time.perf_counter() - t1 > cpu_budget:
        raise TimeoutError
    return O.chi2(dss, w.expr, p)


t1 = time.perf_counter()
try:
    cpu = pkg.minimize("chi2", dss, w.expr, start, objective_fn=cpu_obj)
    t_cpu = time.perf_counter() - t1
    out.update(cpu_fit_s=t_cpu, cpu_evals=cpu.objective_evaluations, cpu_chi2=cpu.objective_value,
               cpu_params=cpu.best_parameters.values.tolist(),
               max_rel_param_diff=float(np.max(np.abs(gpu.best_parameters.values - cpu.best_parameters.values)
                                               / np.maximum(np.abs(cpu.best_parameters.values), 1e-300))),
               speedup=t_cpu / t_gpu)
except TimeoutError:
    t_cpu = time.perf_counter() - t1
    per = t_cpu / calls["n"]
    out.update(cpu_fit_s_extrapolated=per * gpu.objective_evaluations, cpu_s_per_eval=per,
               cpu_evals_timed=calls["n"], speedup_extrapolated=per * gpu.objective_evaluations / t_gpu)
print(json.dumps(out))
