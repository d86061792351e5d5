"""GPU objective sessions: the drop-in replacement for musr.chi2 / musr.mlh.

A *session* is one (datasets, theory, tau_mu, parameter-vector length) problem
resident on one GPU (or one shard of it on one rank).  Building a session:

1. lowers the theory AST to CUDA (codegen.py) and JIT-compiles it (NVRTC);
2. computes, once, the parameter-independent per-bin streams with the same
   numpy expressions the reference evaluates on every call, so they are
   bit-identical to it:
     * fit interval [first, last] from ``range_mask``      musr.py:98-101
     * errors ``max(1, sqrt(d))``                           musr.py:95-96
     * envelope ``exp(-t / tau_mu)``                        musr.py:162
   and uploads counts/errors/envelope of the in-range bins (``musr_upload``);
3. resolves, per dataset, every error the reference interpreter would raise
   for this parameter-vector length (empty range, map coverage / range,
   literal division by zero, N0/Nbkg index) in the reference's order.

An evaluation (``musr_eval``) launches the objective kernel once with p and
the host-evaluated uniform rows inside the kernel parameters (one GPU; the
sharded NCCL path replays a CUDA graph instead) and reads the per-dataset
results as they land in mapped host memory; the host folds them in dataset
order and maps the first failing dataset to the reference exception.  A call
that repeats the last completed problem is validated and launched in C
(``fast_evaluate``, csrc/musr_pyfast.c); anything else comes through
``session_for``.
"""

from __future__ import annotations

import ctypes as C
import operator
import os
import threading
from collections import OrderedDict
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from .codegen import Lowered, lower
from .theory import (
    Binary,
    Call,
    EvalError,
    Num,
    SlotRef,
    TheoryError,
    TimeVar,
    Unary,
    parse,
)

__all__ = ["DeviceBackend", "Session", "shard_assignment", "session_for", "ErrorTypes"]


# -- exception classes used for raised errors ----------------------------------------

@dataclass
class ErrorTypes:
    """Exception classes raised by the objective.  Default: this package's own
    mirrors; ``install()`` swaps in the host package's (e.g. the reference's
    ``blk.musr.MusrError`` / ``blk.theory.EvalError``) so callers catching those
    keep working."""

    musr: type = None
    eval: type = EvalError


ERRORS = ErrorTypes()


# -- backend: device selection / sharding ------------------------------------------

@dataclass(frozen=True)
class DeviceBackend:
    """Execution backend for the GPU objective (the DKS device selection).

    ``world == 1``: one GPU, no collective.  ``world > 1``: this process is
    rank ``rank``; datasets are split into contiguous, bin-balanced shards.
    The per-dataset results are combined either through ``shared_results``
    -- a host buffer mapped by every rank's process, into which each rank's
    kernel writes its datasets' epoch-tagged results (musr_open_shared; the
    default of ``from_torch_distributed``) -- or by one fp64 ncclAllReduce per
    evaluation inside a CUDA graph (``nccl_id``).  Every rank must call the
    objective with the same datasets and p (SPMD), like the reference's single
    caller.
    """

    device: int = 0
    rank: int = 0
    world: int = 1
    nccl_id: Optional[bytes] = field(default=None, repr=False)
    worker_count: int = 1          # accepted for signature compatibility
    collective: bool = False       # force the NCCL path even for world == 1 (tests)
    # (address, bytes) of the ranks' shared result buffer (shared_result_buffer)
    shared_results: Optional[Tuple[int, int]] = field(default=None, repr=False)

    @property
    def kind(self) -> str:
        return f"B200(device={self.device})" if self.world == 1 else \
            f"B200(device={self.device}, rank={self.rank}/{self.world})"

    @classmethod
    def from_torch_distributed(cls, device: Optional[int] = None,
                               combine: str = "host") -> "DeviceBackend":
        """Build a sharded backend from an initialised torch.distributed group
        (plumbing only).  ``combine="host"``: the ranks share a result buffer
        in host memory (one node); ``"nccl"``: an NCCL unique id is broadcast
        for the in-graph ncclAllReduce."""
        import torch.distributed as dist  # plumbing, not the product

        rank, world = dist.get_rank(), dist.get_world_size()
        if device is None:
            import os

            device = int(os.environ.get("LOCAL_RANK", rank))
        if world == 1:
            return cls(device=device)
        if combine == "host":
            return cls(device=device, rank=rank, world=world,
                       shared_results=shared_result_buffer(dist))
        holder = [None]
        if rank == 0:
            holder[0] = new_nccl_id()
        dist.broadcast_object_list(holder, src=0)
        return cls(device=device, rank=rank, world=world, nccl_id=holder[0])


# Shared result buffers of this process: address -> (mmap, sessions opened on it)
_SHARED: Dict[int, list] = {}
SHARED_RESULT_BYTES = 1 << 22      # 2 slots x 4 words x 8 B x 65536 datasets


def shared_result_buffer(dist, nbytes: int = SHARED_RESULT_BYTES) -> Tuple[int, int]:
    """A zero-filled host buffer mapped by every rank of ``dist``'s group (one
    node): rank 0 creates a /dev/shm file, every rank maps it, and rank 0
    removes the name once all have (the mappings stay).  Returns (address,
    bytes) for DeviceBackend.shared_results."""
    import mmap
    import os
    import uuid

    holder = [f"/dev/shm/musr_b200_{uuid.uuid4().hex}" if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(holder, src=0)
    path = holder[0]
    if dist.get_rank() == 0:
        fd = os.open(path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
        os.ftruncate(fd, nbytes)
    dist.barrier()
    if dist.get_rank() != 0:
        fd = os.open(path, os.O_RDWR)
    mm = mmap.mmap(fd, nbytes, mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
    os.close(fd)
    dist.barrier()
    if dist.get_rank() == 0:
        os.unlink(path)
    addr = C.addressof(C.c_char.from_buffer(mm))
    _SHARED[addr] = [mm, 0]
    return addr, nbytes


def new_nccl_id() -> bytes:
    lib = _lib.load()
    buf = C.create_string_buffer(128)
    path = _lib.nccl_library_path()
    _lib.check(lib.musr_nccl_unique_id(path.encode() if path else None, buf), None,
               "musr_nccl_unique_id")
    return buf.raw


def shard_assignment(n_terms: Sequence[int], world: int) -> List[int]:
    """Rank owning each dataset: contiguous blocks balanced by in-range bins.
    Dataset j goes to floor(world * midpoint_j / total), midpoint_j being the
    cumulative bin count at the centre of dataset j."""
    n = [int(x) for x in n_terms]
    total = sum(n)
    if world <= 1 or total == 0:
        return [0] * len(n)
    out = []
    acc = 0
    for x in n:
        mid2 = 2 * acc + x      # 2 * midpoint, integers only
        out.append(min(world - 1, (world * mid2) // (2 * total)))
        acc += x
    return out


# -- per-dataset preparation --------------------------------------------------------

def _adopt_ast(expr):
    """Accept a TheoryExpr from this package or from the reference package:
    rebuild its AST with this package's node classes (same names/fields)."""
    def conv(n):
        name = type(n).__name__
        if name == "Num":
            return Num(float(n.value))
        if name == "TimeVar":
            return TimeVar()
        if name == "SlotRef":
            return SlotRef(str(n.array), int(n.slot))
        if name == "Unary":
            return Unary(n.op, conv(n.operand))
        if name == "Binary":
            return Binary(n.op, conv(n.left), conv(n.right))
        if name == "Call":
            return Call(n.name, tuple(conv(a) for a in n.args))
        raise TypeError(name)

    ast = getattr(expr, "ast", None)
    if ast is not None:
        try:
            return conv(ast)
        except (TypeError, AttributeError):
            pass
    return parse(expr.source).ast


_LOWER_CACHE: Dict[object, Lowered] = {}


def _lowered(ast) -> Lowered:
    low = _LOWER_CACHE.get(ast)
    if low is None:
        low = lower(ast)
        _LOWER_CACHE[ast] = low
    return low


@dataclass
class _Prepared:
    index: int
    detector: int
    error: Optional[BaseException]        # static error for this p length
    first: int = 0
    n_terms: int = 0
    counts: Optional[np.ndarray] = None
    errors: Optional[np.ndarray] = None
    envelope: Optional[np.ndarray] = None


def _static_error(ds, low: Lowered, n_p: int, musr_error: type, eval_error: type):
    """The exception the reference would raise for this dataset *before* the
    MLH positivity check, or None (musr.py:191-197, theory.py:425-435)."""
    m = tuple(ds.binding.map)
    n_f = len(ds.binding.function_values)
    for ev in low.events:
        if ev.kind == "zdiv":
            return ZeroDivisionError("float division by zero")
        k = ev.slot
        if k >= len(m):
            return eval_error(f"slot {k} not covered by map of length {len(m)}")
        j = m[k]
        size = n_p if ev.kind == "p" else n_f
        if j >= size:
            return eval_error(
                f"map entry m[{k}]={j} out of range for {ev.kind!r} array of length {size}"
            )
    for slot in (ds.n0_slot, ds.nbkg_slot):
        if not -n_p <= int(slot) < n_p:
            return IndexError(f"index {int(slot)} is out of bounds for axis 0 with size {n_p}")
    return None


def _prepare(j: int, ds, low: Lowered, tau_mu: float, n_p: int, musr_error, eval_error,
             need_streams: bool) -> _Prepared:
    counts = np.asarray(ds.counts)
    # musr.py:92-93 / 98-101, evaluated exactly as the reference does
    t = (np.arange(len(counts)) - ds.t0_bin) * ds.dt
    lo, hi = ds.fit_range if ds.fit_range is not None else (0.0, np.inf)
    mask = (t >= max(lo, 0.0)) & (t <= hi)
    if not mask.any():
        return _Prepared(j, ds.detector_index,
                         musr_error(f"detector {ds.detector_index}: empty fit range"))
    err = _static_error(ds, low, n_p, musr_error, eval_error)
    if err is not None:
        return _Prepared(j, ds.detector_index, err)
    first = int(np.argmax(mask))
    last = len(mask) - 1 - int(np.argmax(mask[::-1]))
    if not mask[first:last + 1].all():   # t is monotone for dt > 0, so never
        raise ValueError(f"detector {ds.detector_index}: fit range is not contiguous")
    prep = _Prepared(j, ds.detector_index, None, first, last - first + 1)
    if need_streams:
        sl = slice(first, last + 1)
        d = counts.astype(np.float64, copy=False)
        prep.counts = np.ascontiguousarray(d[sl])
        prep.errors = np.ascontiguousarray(np.maximum(1.0, np.sqrt(d))[sl])     # musr.py:95-96
        prep.envelope = np.ascontiguousarray(np.exp(-t / tau_mu)[sl])           # musr.py:162
    return prep


def _fresh(exc: BaseException) -> BaseException:
    """A new instance of a cached static error (clean traceback per raise)."""
    try:
        return type(exc)(*exc.args)
    except Exception:
        return exc


# -- the session ------------------------------------------------------------------------

# Tile shapes (musr_set_tile_shape): 4096-term tiles (8 terms x 16 warps) fill the
# GPU best from ~128 of them on.  A problem of at most SMALL_PROBLEM_TILES such
# tiles (C1: one 2^16-bin histogram = 16 tiles) leaves most SMs idle and is
# latency-bound, so it takes 2048-term tiles of 8 terms x 8 warps: 2^17 bins
# 13.2 -> 11.6 us, 8 x 2^14 bins 18.9 -> 17.4 us -- and up to 16 such tiles
# 1024-term tiles of 8 x 4 warps: C1 chi2 13.2 -> ~11.8 us; at 128 default tiles
# and beyond the default wins (profiles/r2q_ab_tile_shape*.txt).
# The terms per thread stay 8, so every value -- transcendental theories
# included -- is bit-identical to the default shape's, and a rank's choice can
# never make a sharded run differ from the one-GPU run (4 terms per thread was
# ~7 % faster still for C1, but moves transcendental values by an ulp: the
# anchored recurrences restart at each thread's first bin).
SMALL_PROBLEM_TILES = 64


def small_problem_tile_shape(n_terms) -> Optional[Tuple[int, int]]:
    """(terms per thread, consumer warps) for a rank's datasets, or None for
    the default; MUSR_PT / MUSR_CWARPS in the environment take precedence."""
    if "MUSR_PT" in os.environ or "MUSR_CWARPS" in os.environ:
        return None
    tiles = sum(-(-int(n) // 4096) for n in n_terms)
    if tiles <= 0 or tiles > SMALL_PROBLEM_TILES:
        return None
    return (8, 4) if tiles <= SMALL_PROBLEM_TILES // 4 else (8, 8)


class Session:
    """One resident objective problem (see module docstring)."""

    def __init__(self, datasets: Sequence, expr, tau_mu: float, n_p: int,
                 backend: Optional[DeviceBackend] = None, musr_error: type = None,
                 eval_error: type = None):
        self.backend = backend or DeviceBackend()
        self.n_p = int(n_p)
        self.n_global = len(datasets)
        self.tau_mu = float(tau_mu)
        musr_error = musr_error or ERRORS.musr
        eval_error = eval_error or ERRORS.eval
        self.lowered = _lowered(_adopt_ast(expr))
        self._handle = None
        self._lock = threading.Lock()
        lib = _lib.load()

        be = self.backend
        # static analysis for all datasets (every rank knows every dataset's error)
        preps = [_prepare(j, ds, self.lowered, self.tau_mu, self.n_p, musr_error, eval_error,
                          need_streams=False) for j, ds in enumerate(datasets)]
        self.static_errors: List[Tuple[int, BaseException]] = [
            (p.index, p.error) for p in preps if p.error is not None
        ]
        live = [p for p in preps if p.error is None]
        owner = shard_assignment([p.n_terms for p in live], be.world)
        mine = [p for p, r in zip(live, owner) if r == be.rank]
        self.local_indices = [p.index for p in mine]
        self.local_terms = sum(p.n_terms for p in mine)
        self.total_terms = sum(p.n_terms for p in live)
        streams = [_prepare(p.index, datasets[p.index], self.lowered, self.tau_mu, self.n_p,
                            musr_error, eval_error, need_streams=True) for p in mine]

        # per-dataset map / f rows (padded; only validated slots are dereferenced)
        map_stride = max([1, self.lowered.max_p_slot + 1, self.lowered.max_f_slot + 1] +
                         [len(datasets[p.index].binding.map) for p in mine])
        f_stride = max([1] + [len(datasets[p.index].binding.function_values) for p in mine])
        nl = len(mine)
        maps = np.zeros((max(nl, 1), map_stride), dtype=np.int32)
        fvals = np.zeros((max(nl, 1), f_stride), dtype=np.float64)
        n0 = np.zeros(max(nl, 1), dtype=np.int32)
        nbkg = np.zeros(max(nl, 1), dtype=np.int32)
        for i, p in enumerate(mine):
            ds = datasets[p.index]
            m = ds.binding.map
            maps[i, :len(m)] = m
            fv = ds.binding.function_values
            fvals[i, :len(fv)] = fv
            n0[i] = int(ds.n0_slot) % self.n_p       # numpy negative-index wrap
            nbkg[i] = int(ds.nbkg_slot) % self.n_p
        p_capacity = max(1, self.n_p)

        handle = C.c_void_p()
        if be.shared_results is not None:
            addr, nbytes = be.shared_results
            entry = _SHARED.setdefault(addr, [None, 0])
            entry[1] += 1            # sessions are created in the same order on every rank
            _lib.check(lib.musr_open_shared(be.device, be.rank, be.world, C.c_void_p(addr),
                                            nbytes, entry[1] << 24, C.byref(handle)),
                       None, "musr_open_shared")
        elif be.world == 1 and not be.collective:
            _lib.check(lib.musr_open(be.device, C.byref(handle)), None, "musr_open")
        else:
            if be.nccl_id is None or len(be.nccl_id) != 128:
                raise ValueError("sharded DeviceBackend needs a 128-byte nccl_id")
            path = _lib.nccl_library_path()
            _lib.check(lib.musr_open_sharded(be.device, be.rank, be.world,
                                             path.encode() if path else None,
                                             be.nccl_id, C.byref(handle)),
                       None, "musr_open_sharded")
        self._handle = handle
        self._lib = lib
        shape = small_problem_tile_shape([p.n_terms for p in mine])
        self.tile_shape = shape           # None: the library's (8 terms x 16 warps, or env)
        if shape is not None:
            _lib.check(lib.musr_set_tile_shape(handle, *shape), handle, "musr_set_tile_shape")
        log = C.create_string_buffer(1 << 16)
        _lib.check(lib.musr_set_theory(handle, self.lowered.source.encode(), log, len(log)),
                   handle, "musr_set_theory")
        # the parameter-only part as a host program: evaluated per call in C++ like the
        # reference's numpy scalars, passed inline with the launch (small problems)
        ucode = np.ascontiguousarray(self.lowered.uniform_code, dtype=np.int32)
        ulits = np.ascontiguousarray(self.lowered.uniform_lits or [0.0], dtype=np.float64)
        _lib.check(lib.musr_set_uniform_program(handle, ucode.ctypes.data, len(ucode),
                                                ulits.ctypes.data, len(self.lowered.uniform_lits)),
                   handle, "musr_set_uniform_program")

        def arr(a, ct):
            return np.ascontiguousarray(a).ctypes.data_as(C.POINTER(ct))

        out_index = np.array([p.index for p in mine] or [0], dtype=np.int32)
        n_terms = np.array([p.n_terms for p in mine] or [0], dtype=np.int64)
        first_bin = np.array([p.first for p in mine] or [0], dtype=np.int64)
        t0 = np.array([int(datasets[p.index].t0_bin) for p in mine] or [0], dtype=np.int64)
        dts = np.array([float(datasets[p.index].dt) for p in mine] or [0.0], dtype=np.float64)
        keep = [s.counts for s in streams] + [s.errors for s in streams] + \
            [s.envelope for s in streams]
        cptr = (C.c_void_p * max(nl, 1))(*[s.counts.ctypes.data for s in streams])
        eptr = (C.c_void_p * max(nl, 1))(*[s.errors.ctypes.data for s in streams])
        vptr = (C.c_void_p * max(nl, 1))(*[s.envelope.ctypes.data for s in streams])
        rc = lib.musr_upload(
            handle, self.n_global, nl, arr(out_index, C.c_int32), arr(n_terms, C.c_int64),
            arr(first_bin, C.c_int64), arr(t0, C.c_int64), arr(dts, C.c_double),
            C.cast(cptr, C.POINTER(C.c_void_p)), C.cast(eptr, C.POINTER(C.c_void_p)),
            C.cast(vptr, C.POINTER(C.c_void_p)), arr(n0, C.c_int32), arr(nbkg, C.c_int32),
            arr(maps, C.c_int32), map_stride, arr(fvals, C.c_double), f_stride, p_capacity)
        del keep
        _lib.check(rc, handle, "musr_upload")

        self._p = np.zeros(p_capacity, dtype=np.float64)
        self._sums = np.zeros(self.n_global, dtype=np.float64)
        self._bad = np.zeros(self.n_global, dtype=np.int64)
        self._total = np.zeros(1, dtype=np.float64)
        # raw-pointer fast path for the per-evaluation call (see _lib.eval_raw)
        self._eval_raw = _lib.eval_raw()
        self._raw_out = (self._sums.ctypes.data, self._bad.ctypes.data, self._total.ctypes.data)
        self._pview = self._p[:self.n_p]          # per-call staging of p (cached address)
        self._p_addr = self._p.ctypes.data
        self.first_static = self.static_errors[0] if self.static_errors else None

    # -- evaluation ---------------------------------------------------------------
    def run(self, kind: int, p: np.ndarray) -> None:
        """Launch one evaluation; results in self._sums / self._bad / self._total."""
        s, b, t = self._raw_out
        if len(p) == self.n_p:     # copy into the staging vector: cheaper than p.ctypes
            np.copyto(self._pview, p)
            rc = self._eval_raw(self._handle.value, kind, self._p_addr, self.n_p, s, b, t)
        else:
            rc = self._eval_raw(self._handle.value, kind, p.ctypes.data, len(p), s, b, t)
        if rc != _lib.MUSR_OK:
            _lib.check(rc, self._handle, "musr_eval")

    def evaluate(self, kind: int, p, datasets=None, musr_error: type = None) -> float:
        """Objective value with the reference's error semantics.  Calls on one
        session are serialised (the handle and its result buffers are
        single-owner; the reference objectives are pure and thread-safe)."""
        with self._lock:
            return self._evaluate(kind, p, musr_error)

    def _evaluate(self, kind: int, p, musr_error: type = None) -> float:
        p = np.ascontiguousarray(p, dtype=np.float64)
        if len(p) != self.n_p:
            raise ValueError("parameter vector length differs from the session's")
        static = self.first_static
        if static is not None and (static[0] == 0 or self.total_terms == 0):
            raise _fresh(static[1])
        self.run(kind, p)
        if kind == _lib.KIND_MLH:
            bad = np.flatnonzero(self._bad >= 0)
            if len(bad) and (static is None or bad[0] < static[0]):
                j = int(bad[0])
                det = self._detectors[j] if self._detectors is not None else j
                raise (musr_error or ERRORS.musr)(
                    f"detector {det}: model is non-positive at bin {int(self._bad[j])}")
        if static is not None:
            raise _fresh(static[1])
        return float(self._total[0])

    def evaluate_batch(self, kind: int, P, musr_error: type = None) -> np.ndarray:
        """Objective values at every row of ``P`` (n_points x n_p) from one
        pass over the histograms per MUSR_KMAX points (musr_eval_batch).  Row i
        equals ``evaluate(kind, P[i])`` bit for bit; if any row would raise,
        the exception of the first such row (in row order) is raised."""
        with self._lock:
            return self._evaluate_batch(kind, P, musr_error)

    def _evaluate_batch(self, kind: int, P, musr_error: type = None) -> np.ndarray:
        P = np.ascontiguousarray(P, dtype=np.float64)
        if P.ndim != 2 or P.shape[1] != self.n_p:
            raise ValueError("P must be (n_points, n_p) with the session's n_p")
        n = P.shape[0]
        if n == 0:
            return np.zeros(0, dtype=np.float64)
        static = self.first_static
        if static is not None and (static[0] == 0 or self.total_terms == 0):
            raise _fresh(static[1])
        sums = np.empty((n, self.n_global), dtype=np.float64)
        bad = np.empty((n, self.n_global), dtype=np.int64)
        tot = np.empty(n, dtype=np.float64)
        dp = C.POINTER(C.c_double)
        _lib.check(self._lib.musr_eval_batch(
            self._handle, kind, P.ctypes.data_as(dp), n, self.n_p, sums.ctypes.data_as(dp),
            bad.ctypes.data_as(C.POINTER(C.c_int64)), tot.ctypes.data_as(dp)),
            self._handle, "musr_eval_batch")
        if kind == _lib.KIND_MLH:
            for i in range(n):       # first failing point, then its first failing dataset
                hit = np.flatnonzero(bad[i] >= 0)
                if len(hit) and (static is None or hit[0] < static[0]):
                    j = int(hit[0])
                    det = self._detectors[j] if self._detectors is not None else j
                    raise (musr_error or ERRORS.musr)(
                        f"detector {det}: model is non-positive at bin {int(bad[i, j])}")
                if static is not None:
                    break
        if static is not None:
            raise _fresh(static[1])
        self._batch_sums = sums
        return tot

    _detectors: Optional[List[int]] = None
    _frozen: list = []

    def per_dataset(self) -> np.ndarray:
        return self._sums.copy()

    def time_evals(self, kind: int, iters: int, mode: int, flush_l2: int = 0):
        """Device timing (see musr_time_evals): returns ms for modes 0/1 and
        (eval_ms, kernel_ms) for mode 2; mode 3 only flushes (before a call the
        caller times).  flush_l2: 0 none, 1 write a 512 MB buffer before every
        timed launch, 2 that plus a 256 MB read pass (the L2 then holds clean
        lines only)."""
        ms, kms = C.c_double(0.0), C.c_double(0.0)
        _lib.check(self._lib.musr_time_evals(self._handle, kind, iters, mode, int(flush_l2),
                                             C.byref(ms), C.byref(kms)),
                   self._handle, "musr_time_evals")
        return (ms.value, kms.value) if mode == 2 else ms.value

    def data_format(self) -> str:
        """'c32' (compact: fp32 counts + err/rcp table) or 'f64' (fp64 streams)."""
        f, ts = C.c_int(0), C.c_int(0)
        self._lib.musr_format(self._handle, C.byref(f), C.byref(ts))
        return "c32" if f.value == 1 else "f64"

    def launches_per_eval(self) -> int:
        """Kernels of this library per evaluation: the objective kernel, preceded
        by the uniform-table kernel when the local datasets exceed the per-CTA
        staging (64).  0 on a rank without datasets."""
        if self.n_tiles() == 0:
            return 0
        return 1 + (len(self.local_indices) > 64)

    def n_tiles(self) -> int:
        n = C.c_int64(0)
        self._lib.musr_tiles(self._handle, C.byref(n))
        return n.value

    def close(self) -> None:
        if _lib._PYFAST is not None:
            _lib._PYFAST.forget(self)
        _FROZEN.release(self)
        with self._lock:                 # not while another thread evaluates on the handle
            if self._handle:
                self._lib.musr_close(self._handle)
                self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# -- session cache for the drop-in functions ---------------------------------------

_CACHE: "OrderedDict[tuple, Tuple[Session, list]]" = OrderedDict()
_CACHE_MAX = 4
_CACHE_LOCK = threading.Lock()


def _signature(datasets, expr, tau_mu, n_p, backend) -> tuple:
    parts = []
    for ds in datasets:
        fr = ds.fit_range
        fr = None if fr is None else tuple(float(x) for x in fr)   # list / ndarray ranges
        parts.append((id(ds), id(ds.counts), fr, ds.dt, ds.t0_bin, ds.binding,
                      ds.n0_slot, ds.nbkg_slot, ds.detector_index))
    return (tuple(parts), id(expr), getattr(expr, "source", None), tau_mu, n_p, backend)


_FIELDS = operator.attrgetter("counts", "fit_range", "dt", "t0_bin", "binding", "n0_slot",
                              "nbkg_slot", "detector_index")
_LAST = {"datasets": None}
# Bumped by every field assignment on this package's MusrDataset: while it is
# unchanged, a call with the same dataset list (all of this package's class)
# skips the per-field comparison.  (Other dataset types -- the reference's own
# -- are compared field by field on every call.)
DATASET_MUTATIONS = [0]


class _FrozenCounts:
    """Counts arrays held by cached sessions are made read-only.

    The reference reads ``ds.counts`` on every call (musr.py:196); a session
    uploads it once.  So that an in-place edit (``ds.counts[7] += 1``) can never
    be answered from a stale device copy, every counts array a cached session
    was built from is flagged ``writeable = False`` while the session lives:
    the edit raises at the write site.  A caller that re-enables writing
    (``ds.counts.flags.writeable = True``) may edit the array; the next call
    sees the flag, drops the session and rebuilds it from the current
    contents.  Flags are restored when the last session using an array closes.
    """

    def __init__(self):
        self._held: Dict[int, list] = {}        # id(array) -> [array, refs, was_writeable]
        self._of: Dict[int, list] = {}          # id(session) -> arrays it froze
        self._lock = threading.Lock()

    def freeze(self, sess, arrays) -> None:
        mine = []
        with self._lock:
            for a in arrays:
                if not isinstance(a, np.ndarray) or any(a is b for b in mine):
                    continue
                ent = self._held.get(id(a))
                if ent is None or ent[0] is not a:
                    ent = [a, 0, bool(a.flags.writeable)]
                    self._held[id(a)] = ent
                    if ent[2]:
                        try:
                            a.flags.writeable = False
                        except ValueError:
                            pass
                ent[1] += 1
                mine.append(a)
            self._of[id(sess)] = mine
            sess._frozen = mine

    def intact(self, sess) -> bool:
        """No array of ``sess`` was made writable again since it was frozen."""
        for a in sess._frozen:
            if a.flags.writeable:
                return False
        return True

    def release(self, sess) -> None:
        with self._lock:
            for a in self._of.pop(id(sess), ()):
                ent = self._held.get(id(a))
                if ent is None or ent[0] is not a:
                    continue
                ent[1] -= 1
                if ent[1] == 0:
                    del self._held[id(a)]
                    if ent[2] and not a.flags.writeable:
                        try:
                            a.flags.writeable = True
                        except ValueError:
                            pass
            sess._frozen = []


_FROZEN = _FrozenCounts()


def _unchanged(datasets, snaps) -> bool:
    """True when every dataset still has the fields captured in ``snaps``
    (counts compared by identity, the rest by value)."""
    if len(datasets) != len(snaps):
        return False
    try:
        for ds, snap in zip(datasets, snaps):
            if _FIELDS(ds) != snap:
                return False
    except ValueError:   # a replaced counts array compared element-wise
        return False
    return True


def session_for(datasets, expr, tau_mu: float, n_p: int, backend: DeviceBackend) -> Session:
    """Return the cached session for this problem, building it on first use.
    Datasets are treated as immutable while cached; replacing a
    dataset's counts array, fit range or binding invalidates the entry."""
    last = _LAST
    if (last["datasets"] is datasets and last["expr"] is expr and last["tau"] == tau_mu
            and last["n_p"] == n_p and (last["backend"] is backend or last["backend"] == backend)
            and last["ids"] == tuple(map(id, datasets))       # list edited in place
            and ((last["own"] and last["mutations"] == DATASET_MUTATIONS[0])
                 or _unchanged(datasets, last["snaps"]))
            and last["session"]._handle and _FROZEN.intact(last["session"])):
        return last["session"]          # fast path: same call site as last time
    key = _signature(datasets, expr, tau_mu, n_p, backend)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and not _FROZEN.intact(hit[0]):
            # a cached counts array was made writable again (and maybe edited):
            # its device copy can be stale, so rebuild from the current contents
            del _CACHE[key]
            hit[0].close()
            hit = None
        if hit is not None:
            _CACHE.move_to_end(key)
            _remember(datasets, expr, tau_mu, n_p, backend, hit[0])
            return hit[0]
    sess = Session(datasets, expr, tau_mu, n_p, backend)
    sess._detectors = [int(ds.detector_index) for ds in datasets]
    _FROZEN.freeze(sess, [ds.counts for ds in datasets])
    pin = [(ds, ds.counts) for ds in datasets] + [expr]   # keep ids alive while cached
    with _CACHE_LOCK:
        _CACHE[key] = (sess, pin)
        _CACHE.move_to_end(key)
        while len(_CACHE) > _CACHE_MAX:
            _, (old, _) = _CACHE.popitem(last=False)
            old.close()
    _remember(datasets, expr, tau_mu, n_p, backend, sess)
    return sess


def _remember(datasets, expr, tau_mu, n_p, backend, sess) -> None:
    from .musr import MusrDataset

    _LAST.update(datasets=datasets, expr=expr, tau=tau_mu, n_p=n_p, backend=backend,
                 ids=tuple(map(id, datasets)),
                 snaps=[_FIELDS(ds) for ds in datasets], session=sess,
                 own=all(type(ds) is MusrDataset for ds in datasets),
                 mutations=DATASET_MUTATIONS[0])


def fast_evaluate(kind, datasets, expr, p, backend, constants):
    """The objective value when this call repeats the last remembered problem
    (checked in C, musr_pyfast.c), else None: the caller takes session_for."""
    return (_lib._PYFAST or _lib.pyfast()).evaluate(kind, datasets, expr, p, backend, constants)


def fast_remember(sess, datasets, expr, backend, constants) -> bool:
    """Remember a completed call for fast_evaluate.  Sessions with a static
    error are not remembered (their calls raise)."""
    pf = _lib.pyfast()
    if sess.first_static is not None or not sess._handle:
        pf.forget()
        return False
    s, b, t = sess._raw_out
    return pf.remember(sess, datasets, expr, backend, constants, tuple(sess._frozen),
                       sess._handle.value, sess.n_p, sess.n_global, s, b, t, sess._lock)


def clear_cache() -> None:
    if _lib._PYFAST is not None:
        _lib._PYFAST.forget()
    _LAST["datasets"] = None
    with _CACHE_LOCK:
        while _CACHE:
            _, (old, _) = _CACHE.popitem(last=False)
            old.close()
