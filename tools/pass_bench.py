"""Time the FWHT pass kernels alone at one size (for ncu and pass tuning):
optr_rht_encode / optr_rht_decode of one 2^logd vector, per kernel class."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2310_06993_b200 as P
from paper_2310_06993_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--logd", type=int, default=25)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--L", type=int, default=0, help="bucket entries (default 2^logd)")
args = ap.parse_args()
dev = torch.device("cuda", 0)
d = 1 << args.logd
L = args.L or d
x = torch.randn(L, device=dev)
ctx = P.RhtContext.for_length(L, 12345)
y = P.rht_encode(x, ctx)
for _ in range(3):
    P.rht_encode(x, ctx)
torch.cuda.synchronize()
_lib.lib().optr_timing_enable(1)
_lib.timing_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.iters):
    P.rht_encode(x, ctx)
e1.record()
torch.cuda.synchronize()
t = _lib.timing_collect()
ms = e0.elapsed_time(e1) / args.iters
out = {"logd": args.logd, "L": L, "encode_ms": round(ms, 4)}
for k, (tms, n, u) in t.items():
    if n:
        out[k] = {"us_per_launch": round(tms / n * 1e3, 2), "gbs": round(8 * d / (tms / n * 1e-3) / 1e9, 1)}
print(json.dumps(out))
