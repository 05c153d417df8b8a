import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2310_06993_b200.collectives import MaskSpec, tar_allreduce_local
dev = torch.device('cuda', 0)
for n, L in [(2, 5_000_000), (4, 5_000_000), (2, 12_000_000), (2, 25_000_000), (4, 25_000_000), (8, 25_000_000)]:
    g = torch.Generator(device=dev).manual_seed(0)
    xs = [torch.randn(L, device=dev, generator=g) for _ in range(n)]
    mean = sum(x.double() for x in xs) / n
    outs, counts, _ = tar_allreduce_local(xs, rotation=1, ht=True, job_seed=1, generation=1, masks=MaskSpec.none())
    errs = [((o.double() - mean).norm() / mean.norm()).item() for o in outs]
    print(n, L, max(errs), flush=True)
