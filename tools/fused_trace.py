"""Event trace of the fused multi-GPU kernel (torchrun, one rank per GPU):
warm calls, then one traced call; saves gpurun_out/<tag>/trace_r<rank>.npy
(uint32 [grid, cap, 4]: kind<<28|tile, t_begin, t_ready, t_end in ns)."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_06993_b200 import _lib  # noqa: E402
from paper_2310_06993_b200.collectives import MaskSpec  # noqa: E402
from paper_2310_06993_b200.dist import TarCommunicator  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=25_000_000)
ap.add_argument("--tag", default="tr")
ap.add_argument("--cap", type=int, default=256)
ap.add_argument("--steady", type=int, default=0,
                help="trace the last of this many back-to-back async calls (steady state, no barrier skew)")
args = ap.parse_args()
rank = int(os.environ["RANK"])
world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dev = torch.device("cuda", torch.cuda.current_device())
dist.init_process_group("nccl", device_id=dev)
comm = TarCommunicator(max_len=args.L)
x = torch.randn(args.L, device=dev)
out = torch.empty_like(x)
for g in range(4):
    comm.allreduce(x, out, rotation=g % world, ht=True, job_seed=1, generation=g, masks=MaskSpec.coin(g, 0.01))
torch.cuda.synchronize()
dist.barrier()
grid = 148 * 4
buf = torch.zeros(grid * args.cap * 4, dtype=torch.int32, device=dev)
_lib.lib().optr_debug_trace(buf.data_ptr(), args.cap)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if args.steady:
    outs = [torch.empty_like(x) for _ in range(args.steady)]
    _lib.lib().optr_debug_trace(None, 0)
    for g in range(args.steady - 1):
        comm.allreduce(x, outs[g], rotation=g % world, ht=True, job_seed=1, generation=10 + g,
                       masks=MaskSpec.coin(10 + g, 0.01), async_op=True)
    _lib.lib().optr_debug_trace(buf.data_ptr(), args.cap)
e0.record()
comm.allreduce(x, out, rotation=0, ht=True, job_seed=1, generation=9, masks=MaskSpec.coin(9, 0.01),
               async_op=bool(args.steady))
if args.steady:
    comm.join()
e1.record()
torch.cuda.synchronize()
_lib.lib().optr_debug_trace(None, 0)
os.makedirs(f"gpurun_out/{args.tag}", exist_ok=True)
np.save(f"gpurun_out/{args.tag}/trace_r{rank}.npy", buf.view(grid, args.cap, 4).cpu().numpy().view(np.uint32))
print(f"rank {rank} call ms {e0.elapsed_time(e1):.3f}", flush=True)
comm.close()
dist.destroy_process_group()
