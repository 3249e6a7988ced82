"""B200-native data plane for ConServe online/offline co-serving (arXiv 2410.01228).

The hot path -- per-layer forward over a mixed online/offline batch with paged
attention over an HBM block pool, a layer-boundary preemption flag, and
incremental KV checkpoint/restore over the host link -- lives in
libconserve_b200.so (CUDA for sm_100a behind the C-ABI in
include/conserve_b200.h). This package is the thin host-side mirror of the
reference's interface (coserve::KvCacheManager / BatchPlan / SimEngine seams).
"""
from ._ffi import LIB_PATH, CS_PREFILL, CS_DECODE, CS_RECOMPUTE, CS_D2H, CS_H2D  # noqa: F401
from .engine import (  # noqa: F401
    AllocResult, BatchEntry, CsConfigError, CsCudaError, CsError, CsInvalidArgument, CsLogicError, CsPoolError,
    CsRuntimeError, Engine, EvictStats, KvPool, ReleaseStats, ResumeCost, TransferDoneEffects, TransferJob,
    model_config, lib,
)
