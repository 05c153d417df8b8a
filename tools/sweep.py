"""Bucket-size sweep (BASELINE configs[4]): 64 KB .. 1 GB fp32 buckets.

One GPU: n co-resident workers (default 4).  Under torchrun: one worker per
GPU.  Prints one JSON line per size: device ms per allreduce, algBW
(bucket bytes / time, per worker), whole-step roofline fraction, and the
FWHT-pass HBM GB/s.

    python tools/sweep.py [--workers 4] [--max-mb 1024] [--drop 0.01]
    torchrun --nproc-per-node N tools/sweep.py
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import load_peaks, next_pow2, nvlink_peak  # noqa: E402
from paper_2310_06993_b200 import _lib  # noqa: E402
from paper_2310_06993_b200.collectives import MaskSpec, tar_allreduce_local  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=4)
    ap.add_argument("--max-mb", type=float, default=1024)
    ap.add_argument("--drop", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    multi = world > 1
    if multi:
        import torch.distributed as dist

        from paper_2310_06993_b200.dist import TarCommunicator

        dist.init_process_group("nccl", device_id=dev)
    n = world if multi else args.workers
    peaks = load_peaks()
    sizes = []
    mb = 0.0625
    while mb <= args.max_mb:
        sizes.append(int(mb * 1024 * 1024 // 4))
        mb *= 4 if mb < 16 else 2
    comm = TarCommunicator(max_len=max(sizes)) if multi else None
    for L in sizes:
        per_rank = 1 if multi else n
        xs = [torch.randn(L, device=dev) for _ in range(per_rank)]
        outs = [torch.empty_like(x) for x in xs]
        gen = [0]

        def step():
            m = MaskSpec.coin(17 + gen[0], args.drop) if args.drop > 0 else MaskSpec.none()
            if multi:
                comm.allreduce(xs[0], outs[0], rotation=gen[0] % n, ht=True, job_seed=1, generation=gen[0], masks=m)
            else:
                tar_allreduce_local(xs, rotation=gen[0] % n, ht=True, job_seed=1, generation=gen[0], masks=m,
                                    out=outs)
            gen[0] += 1

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        if multi:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        D = next_pow2(L)
        Y = 4 * D
        hbm = per_rank * (8 * L + 3 * Y + Y // n)
        nvl = 2 * Y * (n - 1) // n if multi else 0
        t_roof = max(hbm / (peaks["hbm_gbs"] * 1e9), nvl / (nvlink_peak(n) * 1e9))
        if rank == 0:
            print(json.dumps({"bucket_MB": round(4 * L / 2**20, 4), "entries": L, "dim": D, "workers": n,
                              "gpus": world, "ms": round(ms, 4), "algbw_GBps": round(4 * L / (ms * 1e-3) / 1e9, 2),
                              "busbw_GBps": round(nvl / (ms * 1e-3) / 1e9, 2) if multi else None,
                              "t_roof_ms": round(t_roof * 1e3, 4), "roof_frac": round(t_roof * 1e3 / ms, 4)}),
                  flush=True)
        del xs, outs
        torch.cuda.empty_cache()
    if multi:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
