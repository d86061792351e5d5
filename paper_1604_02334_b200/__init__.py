"""B200-native uSR fit objective (chi2 / maximum log-likelihood).

Drop-in for the objective path of the reference package ``blk``
(``pkg/src/blk/musr.py:181-232``): the theory DSL is parsed on the host,
lowered to CUDA and JIT-compiled with NVRTC for sm_100a; one fused fp64
kernel evaluates model, residual/log-likelihood term and the reference's
pairwise reduction tree, one launch per evaluation with the parameters in the
kernel arguments and the per-dataset results returned through mapped host
memory.  Datasets can be sharded over GPUs (one process per GPU); the ranks
exchange results through a host buffer they all map, or with one fp64 NCCL
all-reduce per evaluation (``combine="nccl"``).

The compute lives in ``libmusr_b200.so`` (C ABI: ``include/musr_b200.h``).
There is no CPU fallback.
"""

from .musr import (  # noqa: F401
    GAMMA_MU,
    OBJECTIVES,
    OBJECTIVES_BATCH,
    TAU_MU_US,
    FitResult,
    MusrDataset,
    MusrError,
    ParameterSet,
    PhysicsConstants,
    chi2,
    chi2_batch,
    default_phases,
    degrees_of_freedom,
    install,
    minimize,
    mlh,
    mlh_batch,
    uninstall,
)
from .objective import DeviceBackend, Session, shard_assignment  # noqa: F401
from .optimize import MinimizeConfig, MinimizeResult, OptimizeError, nelder_mead  # noqa: F401
from .theory import (  # noqa: F401
    EvalError,
    ParseError,
    TheoryBinding,
    TheoryError,
    TheoryExpr,
    parse,
)

__version__ = "0.1.0"
