"""Randomized Hadamard codec on the GPU -- drop-in for ``ubar.hadamard``.

Same names, argument meaning and errors as the reference
(``/root/reference/pkg/src/ubar/hadamard.py``); the arithmetic runs in the
sm_100a kernels of liboptr.so.  Functions accept numpy arrays (copied to the
current CUDA device and back, returning numpy) or CUDA torch tensors
(returning CUDA tensors, enqueued on the current stream).

Numerics: the reference transforms in float64 and the runner casts the wire
to float32 (runner.py:224); here the transform itself runs in float32, which
stays within the north-star 1e-5 relative bound.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import EmptyReceptionError, check, lib

__all__ = [
    "EmptyReceptionError",
    "next_pow2",
    "derive_seed",
    "RhtContext",
    "DropMask",
    "fwht_in_place",
    "rht_encode",
    "rht_decode",
    "mse",
]


def _torch():
    import torch

    return torch


def _is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def next_pow2(n: int) -> int:
    """hadamard.py:25-28."""
    if n <= 1:
        return 1
    return 1 << (int(n) - 1).bit_length()


def derive_seed(job_seed: int, bucket_id: int, generation: int) -> int:
    """hadamard.py:31-34 (SeedSequence port in liboptr, bit-exact)."""
    for v in (job_seed, bucket_id, generation):
        if int(v) < 0 or int(v) >= 1 << 64:
            raise ValueError("seed components must be in [0, 2**64)")
    return int(lib().optr_derive_seed(int(job_seed), int(bucket_id), int(generation)))


def _stream_ptr(t) -> int:
    torch = _torch()
    return torch.cuda.current_stream(t.device).cuda_stream


def _to_device(x, dtype=None):
    """-> (cuda tensor, came_from_numpy)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            raise ValueError("torch tensors must live on a CUDA device")
        t = x.contiguous()
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t, False
    arr = np.ascontiguousarray(np.asarray(x))
    t = torch.from_numpy(arr.astype(np.float32) if arr.dtype != np.float32 else arr)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.cuda(), True


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return _lib.OPTR_F32
    if t.dtype == torch.bfloat16:
        return _lib.OPTR_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


@dataclass(frozen=True)
class RhtContext:
    """hadamard.py:37-55.  ``signs`` is computed on the GPU on first use."""

    dim: int
    seed: int
    orig_len: int
    _cache: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        if not _is_pow2(self.dim):
            raise ValueError(f"dim must be a power of two, got {self.dim}")
        if self.orig_len > self.dim:
            raise ValueError("orig_len exceeds padded dim")
        if not 0 <= int(self.seed) < 1 << 64:
            raise ValueError("seed must be in [0, 2**64)")

    @classmethod
    def for_length(cls, orig_len: int, seed: int) -> "RhtContext":
        return cls(dim=next_pow2(orig_len), seed=seed, orig_len=orig_len)

    def sign_bits(self, device=None):
        """Packed signs on the GPU: int32 tensor, bit k of word k/32 (1 = +1)."""
        torch = _torch()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = str(dev)
        if key not in self._cache:
            words = torch.empty((self.dim + 31) // 32, dtype=torch.int32, device=dev)
            check(lib().optr_rht_signs(words.data_ptr(), self.dim, int(self.seed),
                                       torch.cuda.current_stream(dev).cuda_stream), "rht_signs")
            self._cache[key] = words
        return self._cache[key]

    @property
    def signs(self) -> np.ndarray:
        """float64 +-1 array, like the reference attribute."""
        words = self.sign_bits().cpu().numpy().view(np.uint32)
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[: self.dim]
        return bits.astype(np.float64) * 2.0 - 1.0


@dataclass
class DropMask:
    """Per-entry reception flags for a transformed vector (hadamard.py:58-73)."""

    received: object

    def __post_init__(self):
        torch = _torch()
        if isinstance(self.received, torch.Tensor):
            self.received = self.received.to(torch.bool)
        else:
            self.received = np.asarray(self.received, dtype=bool)

    @property
    def received_count(self) -> int:
        return int(self.received.sum())

    @classmethod
    def full(cls, dim: int) -> "DropMask":
        return cls(np.ones(dim, dtype=bool))


def fwht_in_place(v):
    """Unnormalised Sylvester FWHT (hadamard.py:76-90), float32 on the GPU.
    Mutates ``v`` (numpy or CUDA tensor) and returns it."""
    torch = _torch()
    d = len(v)
    if not _is_pow2(d):
        raise ValueError(f"length must be a power of two, got {d}")
    if isinstance(v, torch.Tensor):
        if not v.is_cuda or v.dtype != torch.float32 or not v.is_contiguous():
            raise ValueError("fwht_in_place needs a contiguous float32 CUDA tensor")
        check(lib().optr_fwht(v.data_ptr(), d, _stream_ptr(v)), "fwht")
        return v
    t, _ = _to_device(v, torch.float32)
    check(lib().optr_fwht(t.data_ptr(), d, _stream_ptr(t)), "fwht")
    v[...] = t.cpu().numpy().astype(v.dtype, copy=False)
    return v


def rht_encode(x, ctx: RhtContext):
    """y = H D pad(x) / sqrt(dim) (hadamard.py:93-102); float32 result."""
    torch = _torch()
    if len(x) != ctx.orig_len:
        raise ValueError(f"expected {ctx.orig_len} entries, got {len(x)}")
    is_t = isinstance(x, torch.Tensor)
    t, from_np = _to_device(x, None if (is_t and x.dtype in (torch.float32, torch.bfloat16)) else torch.float32)
    y = torch.empty(ctx.dim, dtype=torch.float32, device=t.device)
    check(lib().optr_rht_encode(t.data_ptr(), _dtype_code(t), ctx.orig_len, y.data_ptr(), ctx.dim,
                                int(ctx.seed), _stream_ptr(t)), "rht_encode")
    return y.cpu().numpy() if from_np else y


def rht_decode(y_recv, mask: DropMask, ctx: RhtContext):
    """hadamard.py:105-123: zero-fill misses, scale dim/received, inverse,
    truncate.  Raises EmptyReceptionError when nothing arrived (this reads
    the received count back, so it synchronises the stream)."""
    torch = _torch()
    if len(y_recv) != ctx.dim:
        raise ValueError(f"expected {ctx.dim} entries, got {len(y_recv)}")
    if len(mask.received) != ctx.dim:
        raise ValueError("drop mask length does not match dim")
    t, from_np = _to_device(y_recv, torch.float32)
    m = mask.received
    if isinstance(m, torch.Tensor):
        mt = m.to(device=t.device, dtype=torch.uint8).contiguous()
    else:
        mt = torch.from_numpy(np.asarray(m, dtype=np.uint8)).to(t.device)
    out = torch.empty(ctx.orig_len, dtype=torch.float32, device=t.device)
    check(lib().optr_rht_decode(t.data_ptr(), mt.data_ptr(), ctx.dim, ctx.orig_len, int(ctx.seed),
                                out.data_ptr(), _lib.OPTR_F32, _stream_ptr(t)), "rht_decode")
    return out.cpu().numpy() if from_np else out


def mse(a, b) -> float:
    """hadamard.py:126-132 (host helper)."""
    torch = _torch()
    if isinstance(a, torch.Tensor):
        a = a.double().cpu().numpy()
    if isinstance(b, torch.Tensor):
        b = b.double().cpu().numpy()
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"length mismatch: {a.shape} vs {b.shape}")
    return float(np.mean((a - b) ** 2))
