"""Small invocations of every one-GPU kernel family, for compute-sanitizer
(tools/gpu.sh sanitize): the fast plan (strided TMA encode, encode + stage-1
mean, gather decode, strided TMA decode), the general plan (LSU / contiguous
TMA passes, TMA aggregate), RHT off (aggregate + assemble), and the codec
entry points.  Exits non-zero on a CUDA error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2310_06993_b200 as P  # noqa: E402
from paper_2310_06993_b200.collectives import MaskSpec, tar_allreduce_local  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for n, L, ht in [(2, 5_000_000, True), (3, 100_000, True), (4, 50_000, False), (2, 9_000_000, True)]:
    xs = [torch.randn(L, device=dev, generator=g) for _ in range(n)]
    outs, counts, got = tar_allreduce_local(xs, rotation=1, ht=ht, job_seed=1, generation=1,
                                            masks=MaskSpec.coin(3, 0.05), want_received=True)
    torch.cuda.synchronize()
    print(n, L, ht, counts.cpu().tolist())
v = torch.randn(1 << 16, device=dev, generator=g)
P.fwht_in_place(v)
ctx = P.RhtContext.for_length(70_000, 5)
y = P.rht_encode(torch.randn(70_000, device=dev, generator=g), ctx)
x = P.rht_decode(y, P.DropMask(torch.ones(ctx.dim, dtype=torch.bool, device=dev)), ctx)
torch.cuda.synchronize()
print("sanitize case ok")
