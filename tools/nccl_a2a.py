"""NCCL all-to-all / all-gather bus bandwidth, one process per GPU (torchrun)."""
import json
import os

import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
for mb in (64, 256):
    n = mb * (1 << 20) // 4
    x = torch.randn(n, device=dev)
    y = torch.empty_like(x)
    for name, fn in (("all_to_all", lambda: dist.all_to_all_single(y, x)),
                     ("all_gather", lambda: dist.all_gather_into_tensor(y, x[: n // world]))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 * 1e-3
        bus = 4 * n * (world - 1) / world / t / 1e9
        if rank == 0:
            print(json.dumps({"probe": "nccl_" + name, "MB": mb, "world": world, "busbw_GBps": round(bus, 1)}), flush=True)
dist.destroy_process_group()
