"""Benchmark: fp64 chi2 evaluation of the uSR fit objective on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C2|C1|C3|C4] [--objective chi2|mlh]

A *step* is one full objective evaluation: H2D copy of the parameter vector,
uniform-table kernel, objective kernel (model + residual + pairwise tree),
[one fp64 ncclAllReduce when sharded], D2H of the per-dataset results.

* N = 1: the C2 workload (BASELINE.json configs[1]): 8 detector histograms x
  2^20 bins, Gaussian-relaxed TF precession (Eq. 6) with per-detector maps.
* N > 1 (torchrun, one process per GPU): weak scaling -- every rank owns a
  C2-shaped shard (8 datasets x 2^20 bins), all ranks evaluate ONE joint
  chi2 over 8N datasets.  `value` is whole-job bins/s.  The
  ranks' per-dataset results meet in a host buffer they all map (each rank's
  kernel writes its datasets' epoch-tagged results there; no device
  collective); torch.distributed is only the launch / barrier / max plumbing.
  MUSR_BENCH_DEVICE=<d> puts every rank on device d (functional check of the
  N > 1 path on one GPU; gloo plumbing).

`value` (Gbins/s) is device-timed with CUDA events on the library's stream,
inputs resident in HBM, L2 flushed (untimed) before every timed evaluation
(C2 in the compact format is 100 MB < 126 MB L2), max over ranks.  `e2e`
times the public drop-in call `paper_1604_02334_b200.chi2(datasets, expr, p)`
from host numpy p (pinned staging, H2D p, graph replay, D2H results, sync).
`--impl reference` times the reference algorithm's CPU port
(oracle/musr_oracle.py, all host threads) on the same workload.
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

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
TRAFFIC_FILE = ROOT / "profiles" / "roofline_traffic.json"
FALLBACK_HBM_GBS = 6650.0             # B200_PROFILING.md fallback
# algorithmic bytes and FP64 instructions per bin (direct evaluation)
ALG_BYTES_PER_BIN = 16
ALG_FP64_PER_BIN = {"C1": {"chi2": 82, "mlh": 116}, "C2": {"chi2": 84, "mlh": 118},
                    "C3": {"chi2": 204, "mlh": 238}, "C4": {"chi2": 84, "mlh": 118}}


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


def build_workload(name: str, rank: int, world: int):
    from paper_1604_02334_b200 import workloads as W

    if name in ("C2", "C5"):
        w = W.c2(n_hist=8 * world)          # weak scaling: 8 datasets per rank
    elif name == "C4":
        w = W.c4()                          # strong scaling: 64 x 2^22 over all ranks
    elif name == "C3":
        w = W.c3()
    else:
        w = W.c1()
    return w, W.synthesize(w)


def cpu_reference(args, w, dss, budget_s: float, workers: int):
    """Reference algorithm (CPU port) on a bounded sample of the workload."""
    from oracle import musr_oracle as O

    fn = O.chi2 if args.objective == "chi2" else O.mlh
    sample = dss[:1]                         # one dataset (2^20 bins for C2)
    bins = sum(len(d.counts) for d in sample)
    fn(sample, w.expr, w.params, workers=workers)        # warm-up
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        fn(sample, w.expr, w.params, workers=workers)
        times.append(time.perf_counter() - t0)
    return bins, times


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w, dss = build_workload(args.workload, 0, world)
    from oracle import musr_oracle as O

    workers = O.cpu_threads()
    fn = O.chi2 if args.objective == "chi2" else O.mlh
    sample = dss[:1]
    bins = sum(len(d.counts) for d in sample)
    for _ in range(args.warmup):
        fn(sample, w.expr, w.params, workers=workers)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn(sample, w.expr, w.params, workers=workers)
    dt = time.perf_counter() - t0
    value = bins * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "Gbins/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Poisson counts around the workload model)",
        "config": workload_config(args, w, world),
        "cpu_baseline": {"value": value, "unit": "Gbins/s", "cores": workers, "kind": "port",
                         "sample": f"{args.objective} of 1 of {len(dss)} datasets ({bins} bins) per step, "
                                   f"oracle/musr_oracle.py with {workers} map_reduce workers"},
        "e2e": {"value": value, "unit": "Gbins/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(args):
    return f"fp64_{args.objective}_gbins_per_s"


def workload_config(args, w, world):
    return {"workload": args.workload, "objective": args.objective,
            "datasets": w.n_hist, "bins_per_dataset": w.nbins,
            "theory": w.expr.source,
            "parallelism": f"dp{world} (dataset shards; results combined in a host buffer mapped by "
                           f"all ranks, no device collective)" if world > 1 else "single GPU",
            "l2": "flushed before every timed evaluation (untimed)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", default="C2", choices=("C1", "C2", "C3", "C4"))
    ap.add_argument("--objective", default="chi2", choices=("chi2", "mlh"))
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
            dist.init_process_group("gloo")
        backend = pkg.DeviceBackend.from_torch_distributed(local)
    else:
        backend = pkg.DeviceBackend(device=local)

    w, dss = build_workload(args.workload, rank, world)
    kind = _lib.KIND_CHI2 if args.objective == "chi2" else _lib.KIND_MLH
    call = pkg.chi2 if args.objective == "chi2" else pkg.mlh
    total_bins = sum(len(d.counts) for d in dss)
    value0 = call(dss, w.expr, w.params, backend)                 # builds the session (JIT, upload)
    sess = objective.session_for(dss, w.expr, pkg.TAU_MU_US, len(w.params), backend)
    local_bins = sess.local_terms

    def barrier():
        if dist is not None:
            dist.barrier()
        import torch

        torch.cuda.synchronize(local)

    # ---- device-timed throughput -------------------------------------------------
    sess.time_evals(kind, args.warmup, 2, True)
    barrier()
    with ClockSampler(local) as clocks:
        ms, kms = sess.time_evals(kind, args.steps, 2, True)
    barrier()
    if dist is not None:
        import torch

        t = torch.tensor([ms, kms], dtype=torch.float64,
                         device=f"cuda:{local}" if same_device is None else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = t.tolist()
    value = total_bins * args.steps / (ms * 1e-3) / 1e9            # whole job, Gbins/s
    evals_per_s = args.steps / (ms * 1e-3)

    # ---- end to end through the public API (host p, sync per call) ------------------
    p = w.params.copy()
    e2e_times = []
    for i in range(args.warmup + args.steps):
        sess.time_evals(kind, 1, 3, True)      # L2 flush only, outside the timed call
        barrier()
        t0 = time.perf_counter()
        v = call(dss, w.expr, p, backend)
        t1 = time.perf_counter()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
        assert v == value0
    e2e_s = sum(e2e_times)
    if dist is not None:
        import torch

        t = torch.tensor([e2e_s], dtype=torch.float64,
                         device=f"cuda:{local}" if same_device is None else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    e2e_value = total_bins * len(e2e_times) / e2e_s / 1e9

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the objective kernel ------------------------------------------------
    peaks = json.loads(PEAKS_FILE.read_text()) if PEAKS_FILE.exists() else {}
    hbm_peak = peaks.get("hbm_gbs", FALLBACK_HBM_GBS)
    kernel_s = kms * 1e-3 / args.steps
    alg_bytes = ALG_BYTES_PER_BIN * local_bins
    fp64_peak_tflops = _lib.fp64_peak_tflops(local)                # measured DFMA probe
    fp64_instr_peak = fp64_peak_tflops / 2.0                       # T FP64 instr/s (DFMA = 2 flop)
    fp64_alg = ALG_FP64_PER_BIN[args.workload][args.objective] * local_bins / kernel_s / 1e12
    traffic, prof = None, None
    if TRAFFIC_FILE.exists():
        tr = json.loads(TRAFFIC_FILE.read_text())
        prof = tr.get(f"{args.workload}/{args.objective}")
        if prof is not None and world == 1:
            traffic = prof["dram_bytes_per_launch"]
    roofline = {
        "bound": "hbm", "achieved": alg_bytes / kernel_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
        "frac": alg_bytes / kernel_s / 1e9 / hbm_peak, "traffic": traffic,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback",
        "kernel": f"musr_{args.objective}_{sess.data_format()}",
        "kernel_us": kernel_s * 1e6, "alg_bytes_per_bin": ALG_BYTES_PER_BIN,
        "binding": "fp64 (SURVEY.md 8(d))",
        "fp64": {"achieved": fp64_alg, "peak": fp64_instr_peak, "unit": "T fp64 instr/s",
                 "frac": fp64_alg / fp64_instr_peak,
                 "alg_instr_per_bin": ALG_FP64_PER_BIN[args.workload][args.objective],
                 "peak_source": f"measured DFMA probe ({fp64_peak_tflops:.1f} TFLOP/s)"},
    }
    if prof is not None:
        # what the kernel actually executes (ncu: DADD+DMUL+DFMA thread instructions
        # per bin, profiles/roofline_traffic.json) at this run's kernel time
        ex = prof["fp64_thread_inst_per_bin"] * local_bins / kernel_s / 1e12
        roofline["fp64"]["executed"] = {
            "achieved": ex, "frac": ex / fp64_instr_peak,
            "instr_per_bin": prof["fp64_thread_inst_per_bin"],
            "ncu_fp64_pipe_active_pct": prof["fp64_pipe_active_pct"],
            "ncu_issue_active_pct": prof["issue_active_pct"], "source": prof["source"]}

    # ---- CPU baseline (reference algorithm port, bounded sample) --------------------------
    from oracle import musr_oracle as O

    cpu_bins, cpu_times = cpu_reference(args, w, dss, args.cpu_budget, 1)
    cpu_value = cpu_bins * len(cpu_times) / sum(cpu_times) / 1e9

    line = {
        "metric": metric_name(args), "value": value, "unit": "Gbins/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.workload != "C4" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Poisson counts around the workload model; no datasets)",
        "config": workload_config(args, w, world),
        "evals_per_s": evals_per_s, "value_check": value0,
        "e2e": {"value": e2e_value, "unit": "Gbins/s", "evals_per_s": len(e2e_times) / e2e_s,
                "us_per_call": 1e6 * e2e_s / len(e2e_times),
                # p travels in the kernel parameters; results come back as 4
                # epoch-tagged 8-byte words per dataset (all ranks' datasets
                # land in the shared host buffer when sharded)
                "h2d_bytes_per_step": 8 * len(p),
                "d2h_bytes_per_step": 32 * len(dss),
                "api": f"paper_1604_02334_b200.{args.objective}(datasets, expr, p) (reference signature)"},
        "roofline": roofline,
        "cpu_baseline": {"value": cpu_value, "unit": "Gbins/s", "cores": 1, "kind": "port",
                         "sample": f"{len(cpu_times)} x {args.objective} of 1 dataset "
                                   f"({cpu_bins} bins), oracle/musr_oracle.py, 1 thread"},
        # objective-kernel launches inside the two timed regions (K device-timed
        # evaluations + K end-to-end calls); the L2 flushes run outside them
        "gpu_launches": 2 * args.steps,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
