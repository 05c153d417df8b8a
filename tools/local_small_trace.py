"""Phase stamps of the one-GPU small-bucket kernel (n co-resident workers):
device us per call back to back, and CTA 0's phase boundaries (us after
start) for one call.  python tools/local_small_trace.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_06993_b200 import _lib  # noqa: E402
from paper_2310_06993_b200.collectives import MaskSpec, tar_allreduce_local  # noqa: E402

dev = torch.device("cuda", 0)
for n in (4, 8):
    for L in (1 << 14, 1 << 16, 1 << 18, 1 << 20):
        xs = [torch.randn(L, device=dev) for _ in range(n)]
        outs = [torch.empty_like(x) for x in xs]
        m = MaskSpec.coin(5, 0.01)

        def call(g):
            tar_allreduce_local(xs, rotation=g % n, ht=True, job_seed=1, generation=g, masks=m, out=outs)

        for g in range(5):
            call(g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for g in range(100):
            call(g)
        e1.record()
        torch.cuda.synchronize()
        tr = torch.zeros(16, dtype=torch.int64, device=dev)
        _lib.lib().optr_debug_trace(tr.data_ptr(), -1)
        call(7)
        torch.cuda.synchronize()
        _lib.lib().optr_debug_trace(None, -1)
        t = tr.cpu().tolist()
        print(json.dumps({"n": n, "entries": L, "us_per_call": round(e0.elapsed_time(e1) * 10, 2),
                          "phase_us": [round((v - t[0]) / 1e3, 2) for v in t[1:7]]}), flush=True)
