"""Transpose AllReduce with the RHT codec fused in, on the GPU.

Drop-in for ``ubar.collectives`` / ``ubar.schedule`` / ``ubar.wire``
(``/root/reference/pkg/src/ubar/``).  The reference expresses a collective
as a sans-IO generator driven by a channel: those generators (tar, tar2d,
ring, ps) and drivers (``run_lossless``, ``run_datagram``) are re-exported
from ``protocol`` with device buffers and liboptr arithmetic.  The gradient
hot path batches a whole generation instead: the channel is HBM (n workers
on one GPU, ``tar_allreduce_local``) or NVLink (one worker per GPU,
``paper_2310_06993_b200.dist``), and the lossy transport is replaced by
seeded per-packet drop masks (``MaskSpec``) that reproduce the reference's
masks bit-exactly.

Host-side index math (shards, owners, schedule) is plain Python here and is
mirrored in the CUDA kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .protocol import (  # noqa: F401  the reference's sans-IO protocol (collectives.py:25-401)
    AllReduceResult,
    AwaitStage,
    CollectiveDeadlock,
    NodeStats,
    OpenStage,
    RoundEnd,
    SendShard,
    StageResult,
    _mean_received,
    ps_allreduce,
    ring_allreduce,
    run_datagram,
    run_lossless,
    tar2d_allreduce,
    tar_allreduce,
)
from .schedule import PairSchedule, Topology, build_schedule, owned_shard, shard_owner  # noqa: F401

ENTRY_BYTES = 4  # wire.py:23
MAX_PAYLOAD = 1400  # wire.py:22


# ----------------------------------------------------------- index helpers
def shard_lengths(length: int, n: int) -> list[int]:
    """wire.py:121-126."""
    if n < 1:
        raise ValueError("node count must be >= 1")
    base, extra = divmod(int(length), n)
    return [base + 1 if j < extra else base for j in range(n)]


def shard_offsets(length: int, n: int) -> list[int]:
    """wire.py:129-133."""
    offs = [0]
    for ln in shard_lengths(length, n):
        offs.append(offs[-1] + ln)
    return offs


def n_packets(n_entries: int, epp: int) -> int:
    """wire.py:176-180."""
    return -(-int(n_entries) // epp) if n_entries > 0 else 0


# ------------------------------------------------------------------- masks
def mask_words(dim: int, n: int, epp: int) -> int:
    return int(lib().optr_mask_words(int(dim), int(n), int(epp)))


def pack_packet_masks(packets: dict, dim: int, n: int, epp: int) -> np.ndarray:
    """{(stage 1|2, dst, src): bool[n_packets]} -> u32 words in the optr.h
    bitmap layout."""
    pw = mask_words(dim, n, epp)
    words = np.zeros((2, n, n, pw), dtype=np.uint32)
    for (stage, dst, src), pk in packets.items():
        pk = np.asarray(pk, dtype=bool)
        padded = np.zeros(pw * 32, dtype=bool)
        padded[: len(pk)] = pk
        words[stage - 1, dst, src] = np.packbits(padded, bitorder="little").view(np.uint32)
    return words.reshape(-1)


def unpack_packet_masks(words: np.ndarray, dim: int, n: int, r: int, epp: int) -> dict:
    """Inverse of pack_packet_masks (for tests / stats)."""
    pw = mask_words(dim, n, epp)
    w = np.asarray(words, dtype=np.uint32).reshape(2, n, n, pw)
    lens = shard_lengths(dim, n)
    out = {}
    for stage in (1, 2):
        for dst in range(n):
            for src in range(n):
                if src == dst:
                    continue
                j = owned_shard(dst, r, n) if stage == 1 else owned_shard(src, r, n)
                npk = n_packets(lens[j], epp)
                bits = np.unpackbits(w[stage - 1, dst, src].view(np.uint8), bitorder="little")
                out[(stage, dst, src)] = bits[:npk].astype(bool)
    return out


def coin_packets(seed: int, src: int, start: int, count: int, drop_prob: float) -> np.ndarray:
    """Delivered flags of packets ``start .. start+count-1`` of sender ``src``'s
    datagram coin stream (datagram.py:70-72,122), counter-indexed."""
    keep = np.zeros(max(int(count), 0), dtype=np.uint8)
    check(lib().optr_coin_packets(int(seed), int(src), int(start), int(count), float(drop_prob),
                                  keep.ctypes.data if count > 0 else None), "coin_packets")
    return keep.astype(bool)


def coin_masks_host(dim: int, n: int, r: int, seed: int, drop_prob: float,
                    epp: int = MAX_PAYLOAD // ENTRY_BYTES) -> dict:
    """The datagram coin (datagram.py:70-72,117-124) computed by liboptr's host
    port; returns {(stage, dst, src): bool[n_packets]}."""
    pw = mask_words(dim, n, epp)
    buf = np.zeros(2 * n * n * pw, dtype=np.uint32)
    check(lib().optr_masks_host(buf.ctypes.data, int(dim), int(n), int(r), int(seed),
                                float(drop_prob), int(epp)), "masks_host")
    return unpack_packet_masks(buf, dim, n, r, epp)


@dataclass
class MaskSpec:
    """Which packets the lossy channel delivers.

    * ``none``   -- lossless (collectives.py:321-401 run_lossless);
    * ``coin``   -- the UDP backend's seeded send-side coin, sender ``src``
      drawing from ``PCG64(SeedSequence([seed, src]))`` per packet in send
      order (datagram.py:70-72,122), evaluated counter-indexed on the GPU;
    * ``bitmap`` -- explicit per-packet flags, e.g. simulator masks captured
      at consumption time (adaptive-timeout cut-offs, late landings).
    """

    kind: str = "none"
    epp: int = MAX_PAYLOAD // ENTRY_BYTES
    seed: int = 0
    drop_prob: float = 0.0
    bitmap: object = None  # CUDA int32 tensor in the optr.h layout
    # coin: draws each sender's stream made before this call (a reused
    # DatagramEndpoint continues its generator, datagram.py:70-72); None = 0
    stream_offsets: object = None

    @classmethod
    def none(cls, max_payload: int = MAX_PAYLOAD) -> "MaskSpec":
        return cls("none", epp=max_payload // ENTRY_BYTES)

    @classmethod
    def coin(cls, seed: int, drop_prob: float, max_payload: int = MAX_PAYLOAD,
             stream_offsets=None) -> "MaskSpec":
        if not 0.0 <= drop_prob <= 1.0:
            raise ValueError("drop_prob must be in [0,1]")
        offs = None if stream_offsets is None else [int(v) for v in stream_offsets]
        return cls("coin", epp=max_payload // ENTRY_BYTES, seed=int(seed), drop_prob=float(drop_prob),
                   stream_offsets=offs)

    @classmethod
    def from_packets(cls, packets: dict, dim: int, n: int, max_payload: int = MAX_PAYLOAD,
                     device=None) -> "MaskSpec":
        import torch

        epp = max_payload // ENTRY_BYTES
        words = pack_packet_masks(packets, dim, n, epp)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = torch.from_numpy(words.view(np.int32)).to(dev)
        return cls("bitmap", epp=epp, bitmap=t)

    def to_c(self) -> _lib.optr_mask_spec:
        kinds = {"none": _lib.OPTR_MASK_NONE, "coin": _lib.OPTR_MASK_COIN, "bitmap": _lib.OPTR_MASK_BITMAP}
        if self.kind not in kinds:
            raise ValueError(f"unknown mask kind {self.kind!r}")
        if self.epp <= 0:
            raise ValueError("max_payload must hold at least one entry")
        offs = None
        if self.stream_offsets is not None:
            self._offs_c = (ctypes.c_uint64 * _lib.MAX_WORKERS)(*self.stream_offsets)  # kept alive with the spec
            offs = ctypes.addressof(self._offs_c)
        return _lib.optr_mask_spec(kinds[self.kind], int(self.epp), int(self.seed), float(self.drop_prob),
                                   self.bitmap.data_ptr() if self.bitmap is not None else None, offs)


# -------------------------------------------------------- n workers, 1 GPU
_WS: dict = {}
_SLOT: dict = {}
_RETIRED: list = []  # grown-out async workspaces, kept alive until local_join()


def _workspace(n: int, L: int, ht: bool, epp: int, device, key):
    """Cached workspace per (device, caller stream) for synchronous calls and
    per (device, slot) for async calls, so calls on different streams never
    share one."""
    import torch

    need = int(lib().optr_tar_local_workspace(n, L, int(ht), epp))
    ws = _WS.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None and key[1] == "slot":
            _RETIRED.append(ws)  # a queued async call may still use it
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws, need


def local_join(stream=None):
    """Make ``stream`` (default: current) wait for every async
    ``tar_allreduce_local(..., async_op=True)`` call."""
    import torch

    st = stream if stream is not None else torch.cuda.current_stream()
    check(lib().optr_local_join(st.cuda_stream), "local_join")
    # workspaces replaced while async calls were queued: the caller's stream
    # now waits for those calls, so the blocks may return to the allocator
    _RETIRED.clear()


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return _lib.OPTR_F32
    if t.dtype == torch.bfloat16:
        return _lib.OPTR_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


def tar_allreduce_local(buckets: list, *, rotation: int = 0, ht: bool = False, job_seed: int = 0,
                        generation: int = 0, bucket_id: int | None = None,
                        masks: MaskSpec | None = None, out: list | None = None,
                        out_dtype=None, want_received: bool = False, stream=None,
                        async_op: bool = False):
    """One TAR(+RHT) generation for ``n = len(buckets)`` workers whose buckets
    all live on one GPU (the reference's SimSession shape, runner.py:211-276
    with the channel replaced by ``masks``).

    Returns ``(outs, counts, got)``: per-worker output tensors, a CUDA u64
    tensor ``[2, n]`` of received entries per (stage, dst), and (if
    ``want_received``) the ``[n, dim]`` bool AllReduceResult.received.
    Everything is enqueued on ``stream`` (default: current); no host sync.
    ``async_op=True``: the call runs on one of two library streams (two
    buckets in flight); ``out`` and ``counts`` are ready only after
    ``local_join()``; keep every tensor passed in or returned alive and
    untouched until then (``want_received`` needs a synchronous call).
    ``bucket_id`` defaults to ``generation % 65536`` like the runner
    (runner.py:219-222); the RHT seed is derive_seed(job_seed, bucket_id,
    generation).
    """
    import torch

    n = len(buckets)
    if n < 2 or n > _lib.MAX_WORKERS:
        raise ValueError("need 2..16 workers")
    L = len(buckets[0])
    dev = buckets[0].device
    if not buckets[0].is_cuda:
        raise ValueError("buckets must be CUDA tensors")
    for b in buckets:
        if len(b) != L or b.device != dev or b.dtype != buckets[0].dtype or not b.is_contiguous():
            raise ValueError("buckets must be contiguous, same length, dtype and device")
    if async_op and want_received:
        raise ValueError("want_received needs a synchronous call (the flags are converted on the stream)")
    masks = masks or MaskSpec.none()
    out_dtype = out_dtype or buckets[0].dtype
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    dim = (1 << max(0, (L - 1).bit_length())) if ht else L
    # outputs are allocated on the stream the library call is ordered after
    with torch.cuda.stream(st):
        if out is None:
            out = [torch.empty(L, dtype=out_dtype, device=dev) for _ in range(n)]
        # every entry is written by the call (L > 0)
        counts = (torch.empty if L > 0 else torch.zeros)((2, n), dtype=torch.int64, device=dev)
        got = torch.empty((n, dim), dtype=torch.uint8, device=dev) if want_received else None
    xs = (ctypes.c_void_p * n)(*[b.data_ptr() for b in buckets])
    os_ = (ctypes.c_void_p * n)(*[o.data_ptr() for o in out])
    spec = masks.to_c()
    args = (xs, os_, n, L, _dtype_code(buckets[0]), _dtype_code(out[0]), int(job_seed),
            int(generation % 65536 if bucket_id is None else bucket_id), int(generation), int(rotation),
            int(bool(ht)), ctypes.byref(spec))
    if async_op:
        # two in-flight buckets: alternate slots (and their workspaces)
        key = str(dev)
        slot = _SLOT.get(key, 0)
        _SLOT[key] = slot ^ 1
        ws, need = _workspace(n, L, ht, masks.epp, dev, (key, "slot", slot))
        check(lib().optr_tar_local_async(*args, ws.data_ptr(), need, counts.data_ptr(), None, slot, st.cuda_stream),
              "tar_allreduce_local")
    else:
        ws, need = _workspace(n, L, ht, masks.epp, dev, (str(dev), "stream", st.cuda_stream))
        check(lib().optr_tar_local(*args, ws.data_ptr(), need, counts.data_ptr(),
                                   got.data_ptr() if got is not None else None, st.cuda_stream),
              "tar_allreduce_local")
        if got is not None:
            with torch.cuda.stream(st):
                got = got.bool()
    return out, counts, got


def tar_allreduce_batch(entries: list, *, r: int = 0, masks: MaskSpec | None = None) -> list:
    """``tar_allreduce`` (collectives.py:97-150) for all n nodes at once in
    one batched launch sequence, on their already-encoded vectors (RHT is the
    runner's job, runner.py:219-258): stage-1 masked fp64 mean at each shard
    owner, stage-2 assembly.  ``entries``: n equal-length CUDA float32
    tensors; ``masks`` replaces the channel.  Returns one
    ``AllReduceResult(entries, received)`` per node, bit-exact with the
    reference (the generator form is ``tar_allreduce``)."""
    outs, _counts, got = tar_allreduce_local(entries, rotation=r, ht=False, masks=masks, want_received=True)
    return [AllReduceResult(entries=o, received=g) for o, g in zip(outs, got)]


def expected_counts(dim: int, n: int, r: int) -> np.ndarray:
    """[2, n] expected entries per (stage, dst) (simdriver.py:245-248)."""
    lens = shard_lengths(dim, n)
    e = np.zeros((2, n), dtype=np.int64)
    for dst in range(n):
        e[0, dst] = (n - 1) * lens[owned_shard(dst, r, n)]
        e[1, dst] = sum(lens[owned_shard(src, r, n)] for src in range(n) if src != dst)
    return e
