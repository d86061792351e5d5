"""Benchmark: fp64 chi2 (or MLH) evaluations of the uSR fit objective on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C4|C1|C2|C2H|C3] [--objective chi2|mlh] [--combine host|nccl]

The metric (BASELINE.json) is quoted on config C4 -- 64 histograms x 2^22 bins,
Eq. 6 theory, sharded across 1/2/4/8 GPUs -- so C4 is the default workload at
every N (strong scaling: the same 268 M bins split over the ranks).  C1-C3 are
named extra workloads (single GPU); C2H is C2 at N0 = 1e5 (high-statistics
counts, most beyond the count table).  Inputs are the reference generator's
(``blk.musr.generate_synthetic``, SURVEY.md 8(d) seeds and shapes) when the
reference is installed in baseline/_ref, else the package's restatement of it.

A *step* is one full objective evaluation of the whole problem:
  * every rank launches the objective kernel over its shard (p travels in the
    kernel parameters);
  * every rank's host waits until it holds EVERY dataset's result -- all ranks'
    (``--combine host``: the ranks' kernels write their datasets' results into
    one host buffer all ranks map; ``--combine nccl``: one fp64 ncclAllReduce in
    the evaluation's CUDA graph) -- and left-folds the total (musr.py:190-201).
``value`` = total bins x K / (device time of K such steps, max over ranks),
timed with CUDA events on the library's stream around the K steps, after W
untimed ones, bracketed by a barrier and a device sync.  C4 keeps >= 400 MB
per rank (> 126 MB L2) at N <= 8, so its steps run back to back; smaller
workloads flush L2 (512 MB write, untimed) before each step and time each step
with its own events.  ``e2e`` times the public drop-in call
``paper_1604_02334_b200.chi2(datasets, expr, p)`` from a host numpy p (same
rules, host clock).  ``--impl reference`` times the reference's own CPU
objective (``blk.musr.chi2`` from baseline/_ref; the oracle port if absent) on a
bounded sample of the workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REF_DIR = ROOT / "baseline" / "_ref"

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
TRAFFIC_FILE = ROOT / "profiles" / "roofline_traffic.json"
FALLBACK_HBM_GBS = 6650.0             # B200_PROFILING.md fallback
L2_BYTES = 126 << 20
# algorithmic bytes per bin (data d + error err, fp64)
ALG_BYTES_PER_BIN = 16


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled during the timed region."""

    def __init__(self, device: int, period: float = 0.01):
        self.device, self.period = device, period
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap,
                "hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                "hw_power_brake_slowdown": pynvml.nvmlClocksThrottleReasonHwPowerBrakeSlowdown,
            }

            def run():
                while not self._stop.is_set():
                    self.sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    mask = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    self.reasons.update(k for k, v in names.items() if mask & v)
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as exc:  # noqa: BLE001
            self.reasons.add(f"nvml_unavailable:{type(exc).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


# -- workloads ---------------------------------------------------------------------

def reference_package():
    """The unmodified reference (blk) from baseline/_ref, or None."""
    if not (REF_DIR / "blk" / "musr.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import blk.backend
    import blk.musr
    import blk.theory

    return blk


def build_workload(name: str):
    """(Workload, datasets): the reference's generate_synthetic when available
    (shapes, theories, truth = evaluation point, seeds), else
    the package's own synthesis of the same shapes."""
    from paper_1604_02334_b200 import workloads as W

    w = W.WORKLOADS[name]()
    blk = reference_package()
    if blk is None:
        return w, W.synthesize(w), "paper_1604_02334_b200.workloads.synthesize"
    expr = blk.theory.parse(w.expr.source)
    bindings = [blk.theory.TheoryBinding(map=tuple(b.map), function_values=tuple(b.function_values))
                for b in w.bindings]
    truth = blk.musr.ParameterSet(values=w.params.copy(),
                                  names=[f"p{i}" for i in range(len(w.params))],
                                  step_sizes=np.ones(len(w.params)))
    dss = blk.musr.generate_synthetic(truth=truth, expr=expr, bindings=bindings,
                                      n0_slots=w.n0_slots, nbkg_slots=w.nbkg_slots,
                                      nbins=w.nbins, dt=w.dt, seed=w.seed)
    w.expr = expr
    return w, dss, "blk.musr.generate_synthetic (reference, baseline/_ref)"


def needs_flush(w, world: int) -> bool:
    """Flush L2 between timed steps unless each rank streams more than twice
    the L2 (12 B per bin in the compact format); the same rule in both arms, so
    their ``config`` blocks agree."""
    return w.n_hist * w.nbins * 12 / world < 2 * L2_BYTES


def metric_name(args):
    return f"fp64_{args.objective}_gbins_per_s"


def workload_config(args, w, world, flush):
    return {"workload": args.workload, "objective": args.objective,
            "datasets": w.n_hist, "bins_per_dataset": w.nbins,
            "theory": w.expr.source,
            "parallelism": (f"dp{world}: contiguous dataset shards per GPU, per-evaluation "
                            + ("result exchange through a host buffer all ranks map (kernel "
                               "stage-2 stores, no device collective)" if args.combine == "host"
                               else "fp64 ncclAllReduce in the evaluation's CUDA graph"))
            if world > 1 else ("single GPU" if args.combine == "host" else
                               "single GPU, NCCL data plane (1-rank ncclAllReduce in the CUDA graph)"),
            "l2": ("flushed (512 MB write, untimed) before every timed step" if flush else
                   "inputs larger than L2 (no flush; steps back to back)")}


# -- CPU: the reference's own objective on a bounded sample -------------------------------

def cpu_reference_sample(args, w, dss, steps, warmup, budget_s=None):
    """Time the reference CPU objective (blk.musr.chi2 / mlh, Backend(1) and
    Backend(cpu_count), the better one) on one dataset of the workload per
    step.  Falls back to the oracle port when baseline/_ref is absent."""
    sample = dss[:1]
    bins = sum(len(d.counts) for d in sample)
    ncpu = os.cpu_count() or 1
    blk = reference_package()
    if blk is not None:
        fn = blk.musr.chi2 if args.objective == "chi2" else blk.musr.mlh
        p = np.asarray(w.params, dtype=np.float64)
        cands = {k: (lambda b=blk.backend.Backend(worker_count=k): fn(sample, w.expr, p, b))
                 for k in sorted({1, ncpu})}
        kind, what = "reference", f"blk.musr.{args.objective} (baseline/_ref)"
    else:
        from oracle import musr_oracle as O

        fn = O.chi2 if args.objective == "chi2" else O.mlh
        cands = {k: (lambda k=k: fn(sample, w.expr, w.params, workers=k)) for k in sorted({1, ncpu})}
        kind, what = "port", "oracle/musr_oracle.py"
    # choose the faster worker count (the better of Backend(1) / Backend(n))
    probe = {}
    for k, f in cands.items():
        f()
        t0 = time.perf_counter()
        f()
        probe[k] = time.perf_counter() - t0
    best = min(probe, key=probe.get)
    f = cands[best]
    for _ in range(warmup):
        f()
    times = []
    t_end = None if budget_s is None else time.perf_counter() + budget_s
    while len(times) < steps or (t_end is not None and time.perf_counter() < t_end):
        t0 = time.perf_counter()
        f()
        times.append(time.perf_counter() - t0)
        if t_end is not None and len(times) >= steps and time.perf_counter() >= t_end:
            break
    value = bins * len(times) / sum(times) / 1e9
    return {"value": value, "unit": "Gbins/s", "cores": best, "kind": kind,
            "sample": f"{len(times)} x {args.objective} of 1 of {len(dss)} datasets ({bins} bins) "
                      f"per step, {what}, worker_count={best} (probe: "
                      + ", ".join(f"{k}: {1e3 * v:.0f} ms" for k, v in probe.items()) + ")",
            "ms_per_step": 1e3 * sum(times) / len(times)}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w, dss, gen = build_workload(args.workload)
    cb = cpu_reference_sample(args, w, dss, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": metric_name(args), "value": cb["value"], "unit": "Gbins/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if args.workload == "C4" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic: {gen}",
        "config": workload_config(args, w, world, needs_flush(w, world)),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": "Gbins/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -- ours --------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="C4", choices=("C1", "C2", "C2H", "C3", "C4"))
    ap.add_argument("--objective", default="chi2", choices=("chi2", "mlh"))
    ap.add_argument("--combine", default="host", choices=("host", "nccl"),
                    help="multi-GPU result exchange (N > 1)")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of CPU baseline work")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    rank, world, local = dist_env()
    import paper_1604_02334_b200 as pkg
    from paper_1604_02334_b200 import _lib, objective

    dist = None
    same_device = os.environ.get("MUSR_BENCH_DEVICE")
    if same_device is not None:
        local = int(same_device)
    if world > 1:
        import torch
        import torch.distributed as dist  # noqa: F811  (plumbing: rendezvous, barrier, max)

        torch.cuda.set_device(local)
        if same_device is None:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            if args.combine == "nccl":
                raise SystemExit("--combine nccl needs one GPU per rank (NCCL refuses two ranks "
                                 "on one device); MUSR_BENCH_DEVICE checks the host path only")
            dist.init_process_group("gloo")
        backend = pkg.DeviceBackend.from_torch_distributed(local, combine=args.combine)
    elif args.combine == "nccl":   # the NCCL data plane at world 1: graph (kernel + allreduce + D2H)
        backend = pkg.DeviceBackend(device=local, collective=True, nccl_id=objective.new_nccl_id())
    else:
        backend = pkg.DeviceBackend(device=local)

    w, dss, gen = build_workload(args.workload)
    expr = w.expr
    kind = _lib.KIND_CHI2 if args.objective == "chi2" else _lib.KIND_MLH
    call = pkg.chi2 if args.objective == "chi2" else pkg.mlh
    total_bins = sum(len(d.counts) for d in dss)
    p = np.asarray(w.params, dtype=np.float64).copy()
    value0 = call(dss, expr, p, backend)                      # builds the session (JIT, upload)
    sess = objective.session_for(dss, expr, pkg.TAU_MU_US, len(p), backend)
    local_bins = sess.local_terms
    stream_bytes = local_bins * (12 if sess.data_format() == "c32" else 16)
    flush = needs_flush(w, world) or stream_bytes < 2 * L2_BYTES   # C4: >= 400 MB per rank
    launches = sess.launches_per_eval()

    def barrier():
        if dist is not None:
            dist.barrier()
        import torch

        torch.cuda.synchronize(local)

    def max_over_ranks(vals):
        if dist is None:
            return vals
        import torch

        t = torch.tensor(vals, dtype=torch.float64,
                         device=f"cuda:{local}" if same_device is None else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    # ---- value: K synchronous joint evaluations (device clock, max over ranks) -------
    sess.time_evals(kind, args.warmup, 4, flush)
    barrier()
    with ClockSampler(local) as clocks:
        ms = sess.time_evals(kind, args.steps, 4, flush)
    barrier()
    (ms,) = max_over_ranks([ms])
    value = total_bins * args.steps / (ms * 1e-3) / 1e9            # whole job, Gbins/s

    # ---- e2e: the public drop-in call from host numpy p ---------------------------------
    e2e_s = 0.0
    for i in range(args.warmup + args.steps):
        if flush or i == args.warmup:
            sess.time_evals(kind, 1, 3, flush)   # L2 flush (if any) + sync, outside the timing
            barrier()
            t0 = time.perf_counter()
        v = call(dss, expr, p, backend)
        if flush and i >= args.warmup:
            e2e_s += time.perf_counter() - t0
        assert v == value0
    if not flush:
        e2e_s = time.perf_counter() - t0
    barrier()
    (e2e_s,) = max_over_ranks([e2e_s])
    e2e_value = total_bins * args.steps / e2e_s / 1e9

    # ---- the objective kernel alone (roofline): per-launch events -----------------------
    kms = sess.time_evals(kind, args.steps, 1, flush)
    pipe_ms = sess.time_evals(kind, args.steps, 0, 0) if not flush else None
    (kms,) = max_over_ranks([kms])

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks = json.loads(PEAKS_FILE.read_text()) if PEAKS_FILE.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", FALLBACK_HBM_GBS)
    kernel_s = kms * 1e-3 / args.steps
    alg_bytes = ALG_BYTES_PER_BIN * local_bins
    traffic, prof = None, None
    if TRAFFIC_FILE.exists():
        tr = json.loads(TRAFFIC_FILE.read_text())
        prof = tr.get(f"{args.workload}/{args.objective}" + (f"/n{world}" if world > 1 else ""))
        if prof is not None:
            traffic = prof["dram_bytes_per_launch"]
    roofline = {
        "bound": "hbm", "achieved": alg_bytes / kernel_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
        "frac": alg_bytes / kernel_s / 1e9 / hbm_peak, "traffic": traffic,
        "peak_source": "of measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks
                       else "of fallback (B200_PROFILING.md)",
        "kernel": f"musr_{args.objective}_{sess.data_format()}", "kernel_us": kernel_s * 1e6,
        "per_launch_bins": local_bins, "alg_bytes_per_bin": ALG_BYTES_PER_BIN,
        "streamed_bytes_per_bin": stream_bytes / local_bins,
    }
    if traffic is not None:
        # physical DRAM traffic of one launch (ncu dram__bytes_read + write) at this
        # run's kernel time: the bandwidth the kernel actually pulls
        roofline["dram"] = {"achieved": traffic / kernel_s / 1e9, "frac": traffic / kernel_s / 1e9 / hbm_peak,
                            "bytes_per_bin": traffic / local_bins, "source": prof["source"]}
        if "fp64_thread_inst_per_bin" in prof:
            fp64_peak = _lib.fp64_peak_tflops(local) / 2.0        # T DFMA instr/s (probe)
            ex = prof["fp64_thread_inst_per_bin"] * local_bins / kernel_s / 1e12
            roofline["fp64_executed"] = {
                "achieved": ex, "peak": fp64_peak, "unit": "T fp64 instr/s", "frac": ex / fp64_peak,
                "instr_per_bin": prof["fp64_thread_inst_per_bin"],
                "ncu_fp64_pipe_active_pct": prof.get("fp64_pipe_active_pct"),
                "ncu_issue_active_pct": prof.get("issue_active_pct"),
                "peak_source": "measured DFMA probe (musr_fp64_peak)"}

    cpu = cpu_reference_sample(args, w, dss, 2, 1, budget_s=args.cpu_budget)

    line = {
        "metric": metric_name(args), "value": value, "unit": "Gbins/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.workload == "C4" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": f"synthetic: {gen}",
        "config": workload_config(args, w, world, flush),
        "evals_per_s": args.steps / (ms * 1e-3), "value_check": value0,
        "e2e": {"value": e2e_value, "unit": "Gbins/s", "evals_per_s": args.steps / e2e_s,
                "us_per_call": 1e6 * e2e_s / args.steps,
                # p travels in the kernel parameters; results come back as 4
                # epoch-tagged 8-byte words per dataset (all ranks' datasets land
                # in the shared host buffer when sharded)
                "h2d_bytes_per_step": 8 * len(p), "d2h_bytes_per_step": 32 * len(dss),
                "api": f"paper_1604_02334_b200.{args.objective}(datasets, expr, p) "
                       "(reference signature)"},
        "roofline": roofline,
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        # objective launches inside the timed regions: K steps (value), K drop-in
        # calls (e2e), K kernel-timing launches [, K pipelined launches]; the L2
        # flushes run outside them
        "gpu_launches": launches * args.steps * (3 + (pipe_ms is not None)),
        "clocks": clocks.summary(),
    }
    if pipe_ms is not None:
        line["pipelined"] = {"value": local_bins * args.steps / (pipe_ms * 1e-3) / 1e9,
                             "unit": "Gbins/s per rank",
                             "note": "K launches back to back, no host wait between them"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
