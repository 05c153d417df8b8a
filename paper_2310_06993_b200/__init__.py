"""B200-native OptiReduce hot path: RHT encode -> Transpose AllReduce with
masked mean -> masked RHT decode, as sm_100a CUDA kernels behind a C ABI
(include/optr.h, liboptr.so) with a Python facade mirroring the reference
package ``ubar`` (hadamard / collectives / schedule / runner entry points,
the UBT control rules in ``ubt``) and a PyTorch DDP comm hook."""

from ._lib import EmptyReceptionError, LIB_PATH, lib  # noqa: F401
from .collectives import (  # noqa: F401
    AllReduceResult,
    MaskSpec,
    build_schedule,
    owned_shard,
    shard_lengths,
    shard_offsets,
    shard_owner,
    tar2d_allreduce,
    tar_allreduce,
    tar_allreduce_batch,
    tar_allreduce_local,
    ps_allreduce,
    ring_allreduce,
    run_datagram,
    run_lossless,
)
from .schedule import PairSchedule, Topology  # noqa: F401
from .hadamard import (  # noqa: F401
    DropMask,
    RhtContext,
    derive_seed,
    fwht_in_place,
    mse,
    next_pow2,
    rht_decode,
    rht_encode,
)
from .session import GenerationReport, GpuSession  # noqa: F401
