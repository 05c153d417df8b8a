"""Small-bucket latency at N GPUs (torchrun): per bucket size, the device
time per call with R back-to-back async calls, the host issue time per call,
and the library's own per-launch kernel durations (CUDA events around each
launch).  One JSON line per size on rank 0.

    torchrun --nproc-per-node N tools/small_bench.py [--reps 200]
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_06993_b200 import _lib  # noqa: E402
from paper_2310_06993_b200.collectives import MaskSpec  # noqa: E402
from paper_2310_06993_b200.dist import TarCommunicator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--drop", type=float, default=0.01)
    ap.add_argument("--sizes-kb", default="64,256,1024,4096")
    ap.add_argument("--trace", action="store_true", help="small-kernel phase stamps (us after start, median call)")
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    sizes = [int(kb) * 256 for kb in args.sizes_kb.split(",")]
    comm = TarCommunicator(max_len=max(sizes))
    masks = [MaskSpec.coin(17 + g, args.drop) for g in range(8)]
    for L in sizes:
        x = torch.randn(L, device=dev)
        out = torch.empty_like(x)

        def call(g, async_op=True):
            comm.allreduce(x, out, rotation=g % world, ht=True, job_seed=1, generation=g, masks=masks[g % 8],
                           async_op=async_op)

        for g in range(5):
            call(g, False)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for g in range(args.reps):
            call(g)
        h1 = time.perf_counter()
        comm.join()
        e1.record()
        torch.cuda.synchronize()
        dev_us = e0.elapsed_time(e1) / args.reps * 1e3
        host_us = (h1 - h0) / args.reps * 1e6
        # per-launch kernel durations (events around each launch)
        dist.barrier()
        _lib.timing_enable(True)
        for g in range(50):
            call(g, False)
        torch.cuda.synchronize()
        tk = _lib.timing_collect()
        _lib.timing_enable(False)
        kern = {k: round(v[0] / max(v[1], 1) * 1e3, 2) for k, v in tk.items() if v[1]}
        # phase stamps of the small kernel (CTA 0; globaltimer ns)
        phases = None
        if args.trace:
            tr = torch.zeros(64 * 16, dtype=torch.int64, device=dev)
            _lib.lib().optr_debug_trace(tr.data_ptr(), -1)
            for g in range(20):
                call(g, False)
            torch.cuda.synchronize()
            _lib.lib().optr_debug_trace(None, -1)
            rows = tr.view(64, 16).cpu().numpy()
            rows = rows[rows[:, 0] > 0]
            d = (rows[:, 1:] - rows[:, :1]) / 1e3
            phases = [round(float(v), 2) for v in sorted(d.tolist(), key=lambda r: r[-1])[len(d) // 2]]
        t = torch.tensor([dev_us, host_us], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"gpus": world, "bucket_KB": 4 * L // 1024, "entries": L, "drop": args.drop,
                              "device_us_per_call": round(float(t[0]), 2),
                              "host_issue_us_per_call": round(float(t[1]), 2), "kernel_us": kern, "phase_us_rank0": phases}), flush=True)
        del x, out
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
