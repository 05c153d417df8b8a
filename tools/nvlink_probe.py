"""Measure the interconnect peaks the roofline uses, on the GPU box.

Single process over all visible GPUs: copy-engine peer copy, SM pull
(kernel reads a peer buffer), SM push (kernel writes a peer buffer), local
HBM copy; then NCCL all-to-all bus bandwidth with one process per GPU.
Prints one JSON line per measurement.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_06993_b200 import _lib  # noqa: E402

MB = 1 << 20


def timeit(fn, dev, reps=20):
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn(s)
        e1.record(s)
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    n = torch.cuda.device_count()
    lib = _lib.lib()
    nbytes = 512 * MB
    bufs = [torch.empty(nbytes // 4, device=f"cuda:{i}") for i in range(n)]
    for i in range(n):
        for j in range(n):
            if i != j:
                lib.optr_probe_enable_peer(i, j)
    out = []
    d0 = torch.device("cuda:0")
    loc = torch.empty_like(bufs[0])
    t = timeit(lambda s: lib.optr_probe_copy(loc.data_ptr(), bufs[0].data_ptr(), nbytes, 148 * 4, 0, s.cuda_stream), d0)
    out.append({"probe": "hbm_copy_sm", "GBps_rw": round(2 * nbytes / t / 1e9, 1)})
    if n >= 2:
        t = timeit(lambda s: bufs[1].copy_(bufs[0], non_blocking=True), d0)
        out.append({"probe": "peer_copy_engine_0to1", "GBps": round(nbytes / t / 1e9, 1)})
        for blocks in (148, 296, 592, 1184):
            t = timeit(lambda s: lib.optr_probe_copy(loc.data_ptr(), bufs[1].data_ptr(), nbytes, blocks, 0,
                                                     s.cuda_stream), d0)
            out.append({"probe": "sm_pull_1to0", "blocks": blocks, "GBps": round(nbytes / t / 1e9, 1)})
            t = timeit(lambda s: lib.optr_probe_copy(bufs[1].data_ptr(), loc.data_ptr(), nbytes, blocks, 0,
                                                     s.cuda_stream), d0)
            out.append({"probe": "sm_push_0to1", "blocks": blocks, "GBps": round(nbytes / t / 1e9, 1)})
        # every GPU pulls from every peer at once (the TAR exchange pattern):
        # chunks of 16-byte multiples, one stream per (GPU, peer), return codes
        # checked, wall clock around synchronised rounds
        import time

        chunk = (nbytes // (n - 1)) // MB * MB
        locs = [torch.empty(nbytes // 4, device=f"cuda:{i}") for i in range(n)]
        streams = {(i, j): torch.cuda.Stream(torch.device("cuda", i)) for i in range(n) for j in range(n) if i != j}
        blocks = max(1, 148 * 2 // (n - 1))

        def pull_all():
            for i in range(n):
                for k, j in enumerate(p for p in range(n) if p != i):
                    rc = lib.optr_probe_copy(locs[i].data_ptr() + k * chunk, bufs[j].data_ptr(), chunk, blocks, i,
                                             streams[(i, j)].cuda_stream)
                    assert rc == 0, rc
            for i in range(n):
                torch.cuda.synchronize(torch.device("cuda", i))

        for _ in range(3):
            pull_all()
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            pull_all()
        t = (time.perf_counter() - t0) / reps
        out.append({"probe": "sm_pull_all_gpus_all_peers_wallclock", "gpus": n,
                    "GBps_per_gpu_in": round(chunk * (n - 1) / t / 1e9, 1),
                    "note": "every GPU pulls (n-1) chunks from its peers concurrently; wall clock per round"})
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
