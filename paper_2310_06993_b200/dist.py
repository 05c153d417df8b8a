"""One TAR worker per GPU: the multi-GPU drop-in for ``tar_allreduce``.

The reference runs one ``tar_allreduce`` generator per node over a channel
(``/root/reference/pkg/src/ubar/collectives.py:97-150`` driven by
``datagram.py:85-207`` on real sockets).  Here each process owns one GPU and
calls ``TarCommunicator.allreduce`` with its own bucket:

* encode its bucket into its symmetric wire buffer (CUDA-IPC-mapped into
  every peer);
* device barrier (flags over NVLink);
* stage 1: pull its owned shard from every peer's wire buffer over NVLink
  and take the masked fp64 mean (collectives.py:113-125);
* stage 2, fused into the same kernel: the owner pushes its aggregate into
  every peer's symmetric gather buffer over NVLink (collectives.py:127-150);
* device barrier; masked decode from the local gather buffer
  (runner.py:248-256).

That is the barrier path (other sizes).  For D = 2^23..2^25 and n in
{2, 4, 8} the encode's contiguous pass, both stages and the decode's
contiguous pass run in one persistent kernel with per-tile flags over NVLink
(DESIGN.md §5).

torch.distributed (NCCL) only carries the one-time IPC handle exchange and
host barriers; the data path is peer loads inside the kernels.
"""

from __future__ import annotations

import ctypes

from . import _lib
from ._lib import check, lib
from .collectives import MaskSpec


def all_gather_bytes(blob: bytes, group=None, device=None) -> list:
    """Exchange one equal-length byte blob per rank (rank order)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.tensor(list(blob), dtype=torch.uint8)
    if device is not None and dist.get_backend(group) != "gloo":
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return [bytes(p.cpu().tolist()) for p in parts]


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return _lib.OPTR_F32
    if t.dtype == torch.bfloat16:
        return _lib.OPTR_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


class TarCommunicator:
    """Symmetric NVLink buffers for buckets of up to ``max_len`` entries."""

    def __init__(self, max_len: int, epp: int = 350, group=None, device=None, fused_ctas: int = 0):
        import torch
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.max_len = int(max_len)
        self.epp = int(epp)
        h = ctypes.c_void_p()
        check(lib().optr_comm_create(ctypes.byref(h), self.device.index, self.rank, self.world,
                                     self.max_len, self.epp), "comm_create")
        self._h = h
        nb = int(lib().optr_comm_handle_bytes())
        mine = (ctypes.c_char * nb)()
        check(lib().optr_comm_get_handle(self._h, mine), "comm_get_handle")
        blobs = all_gather_bytes(bytes(mine), group, self.device)
        allb = b"".join(blobs)
        check(lib().optr_comm_open(self._h, allb), "comm_open")
        if fused_ctas:
            self.set_fused_ctas(fused_ctas)
        dist.barrier(group)

    def set_fused_ctas(self, ctas: int) -> None:
        """Cap the persistent fused kernel at ``ctas`` CTAs (0 = one per SM x
        occupancy); fewer leave SMs to concurrent work such as DDP's backward
        pass."""
        check(lib().optr_comm_set_fused_grid(self._h, int(ctas)), "comm_set_fused_grid")

    def allreduce(self, x, out, *, rotation: int, ht: bool = True, job_seed: int = 0,
                  generation: int = 0, bucket_id: int | None = None, masks: MaskSpec | None = None,
                  received=None, stream=None, async_op: bool = False, deadline_ns: int = 0,
                  stats=None, cut_units=None):
        """This rank's part of one TAR(+RHT) generation.  ``x``/``out`` are
        this rank's CUDA buffers (fp32/bf16).  ``received``: optional CUDA
        int64[2] for (stage-1, stage-2) received entries.

        ``async_op=True`` lets consecutive buckets overlap (optr_tar_async):
        the stream does not wait for ``out`` until ``join()``; keep ``x`` and
        ``out`` untouched until then.

        ``deadline_ns`` bounds stage 1 (optr_tar_bounded): past it an owner
        aggregates without the peers whose encoded tiles are still missing.
        ``stats``: optional CUDA int64[7] optr_tar_stats (received[2],
        cut[2], t_open, t_stage1, t_stage2 in device-timer ns);
        ``cut_units``: optional CUDA int32 tensor, one word per stage-1 unit
        (bitmask of the peers cut from it)."""
        import torch

        if self._h is None:
            raise RuntimeError("communicator closed")
        if len(x) != len(out) or len(x) > self.max_len:
            raise ValueError("bucket longer than the communicator's max_len")
        masks = masks or MaskSpec.none(self.epp * 4)
        spec = masks.to_c()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        bid = int(generation % 65536 if bucket_id is None else bucket_id)
        if deadline_ns or stats is not None or cut_units is not None:
            if received is not None:
                raise ValueError("pass stats (received counts included) with a deadline")
            check(lib().optr_tar_bounded(self._h, x.data_ptr(), out.data_ptr(), len(x), _dtype_code(x),
                                         _dtype_code(out), int(job_seed), bid, int(generation), int(rotation),
                                         int(bool(ht)), ctypes.byref(spec), int(deadline_ns),
                                         stats.data_ptr() if stats is not None else None,
                                         cut_units.data_ptr() if cut_units is not None else None,
                                         int(bool(async_op)), st.cuda_stream), "tar_bounded")
            return out
        fn = lib().optr_tar_async if async_op else lib().optr_tar
        check(fn(self._h, x.data_ptr(), out.data_ptr(), len(x), _dtype_code(x), _dtype_code(out),
                 int(job_seed), bid, int(generation), int(rotation), int(bool(ht)), ctypes.byref(spec),
                 received.data_ptr() if received is not None else None, st.cuda_stream),
              "tar")
        return out

    def join(self, stream=None):
        """Make ``stream`` (default: current) wait for all async calls."""
        import torch

        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(lib().optr_comm_join(self._h, st.cuda_stream), "comm_join")

    def close(self):
        """Collective: every rank must call it.  No rank unmaps or frees its
        symmetric buffer while a peer's kernels may still read it or store
        flags into it (local drain, then an all-rank barrier)."""
        if self._h is not None:
            import torch
            import torch.distributed as dist

            torch.cuda.synchronize(self.device)
            if dist.is_initialized():
                dist.barrier(self.group)
            lib().optr_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        # no collective barrier from a finaliser: only drain locally
        try:
            if self._h is not None:
                import torch

                torch.cuda.synchronize(self.device)
                lib().optr_comm_destroy(self._h)
                self._h = None
        except Exception:
            pass
