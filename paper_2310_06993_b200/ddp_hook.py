"""PyTorch DDP communication hook: OptiReduce's TAR+RHT as the gradient
all-reduce (PAPER.md:402-419 describes the reference system's hook; the
reference package itself has none).

    state = OptiReduceState(process_group=None, max_bucket_len=..., ht=True)
    ddp_model.register_comm_hook(state, optireduce_hook)

Each DDP bucket (flat fp32 or bf16 gradients) goes through
``TarCommunicator.allreduce`` on the current stream: RHT encode, stage-1
masked mean at the owner, stage-2 receive fused into the decode, one worker
per GPU over NVLink.  The generation counter advances after the last bucket
of every backward pass and the owner rotation follows it
(runner.py:274-275); the RHT seed is derive_seed(seed, bucket.index(),
generation) (hadamard.py:31-34).  NVLink is lossless, so by default nothing is
dropped; ``drop_prob > 0`` emulates the paper's lossy transport with the
seeded datagram coin (per generation and bucket).

The hook enqueues work and returns an already-completed future.  With
``overlap=True`` (default) buckets are enqueued with ``optr_tar_async`` so a
bucket's encode and stage 1 run behind the previous bucket's decode; the
last bucket of the pass joins them onto the reducer's stream.  That is safe
because the reducer copies the hook results back into the gradients only in
its end-of-backward finalisation, after every bucket's hook has run, on the
same stream.  ``overlap=False`` orders every bucket on the stream.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .collectives import MaskSpec
from .hadamard import derive_seed

_COIN_TAG = 0x636F696E  # "coin"


@dataclass
class OptiReduceState:
    process_group: object = None
    max_bucket_len: int = 25 * 1024 * 1024 // 4
    ht: bool = True
    seed: int = 0
    drop_prob: float = 0.0
    max_payload: int = 1400
    generation: int = 0
    overlap: bool = True
    fused_ctas: int = 0  # cap on the fused kernel's CTAs (0 = all SMs); leaves SMs to backward
    comm: object = field(default=None, repr=False)
    received: list = field(default_factory=list, repr=False)  # per-bucket [2] counts of the last pass
    _pending: list = field(default_factory=list, repr=False)  # buffers async calls still use

    def communicator(self, device, needed_len: int = 0):
        """The NVLink communicator, (re)created collectively when a bucket is
        longer than its buffers: every rank sees the same bucket sequence, so
        every rank grows at the same call."""
        if self.comm is not None and needed_len > self.comm.max_len:
            self.comm.close()
            self.comm = None
            self.max_bucket_len = max(needed_len, 2 * self.max_bucket_len)
        if self.comm is None:
            from .dist import TarCommunicator

            self.comm = TarCommunicator(max_len=max(self.max_bucket_len, needed_len),
                                        epp=self.max_payload // 4, group=self.process_group, device=device,
                                        fused_ctas=self.fused_ctas)
        return self.comm

    def masks(self, bucket_index: int) -> MaskSpec:
        if self.drop_prob <= 0.0:
            return MaskSpec.none(self.max_payload)
        seed = derive_seed(self.seed ^ _COIN_TAG, bucket_index, self.generation)
        return MaskSpec.coin(seed, self.drop_prob, self.max_payload)


def max_bucket_len_for(model, bucket_cap_mb: float = 25.0, dtype_bytes: int = 4) -> int:
    """Upper bound on DDP bucket lengths: the reducer closes a bucket once it
    reaches the cap, so a bucket holds less than cap + its last parameter."""
    cap = int(bucket_cap_mb * 1024 * 1024 // dtype_bytes)
    biggest = max((p.numel() for p in model.parameters() if p.requires_grad), default=1)
    return cap + biggest + 1024


def optireduce_hook(state: OptiReduceState, bucket):
    import torch

    buf = bucket.buffer()
    if not buf.is_contiguous():
        buf = buf.contiguous()
    comm = state.communicator(buf.device, buf.numel())
    out = torch.empty_like(buf)
    rec = torch.empty(2, dtype=torch.int64, device=buf.device)  # both entries written by the call
    world = comm.world
    comm.allreduce(buf, out, rotation=state.generation % world, ht=state.ht, job_seed=state.seed,
                   generation=state.generation, bucket_id=bucket.index(), masks=state.masks(bucket.index()),
                   received=rec, async_op=state.overlap)
    if state.overlap:
        # keep every buffer the queued kernels touch alive until the join
        state._pending.append((buf, out, rec))
        if bucket.is_last():
            comm.join()
            state._pending = []
    if bucket.index() == 0:
        state.received = []
    state.received.append(rec)
    if bucket.is_last():
        state.generation += 1
    fut = torch.futures.Future()
    fut.set_result(out)
    return fut
