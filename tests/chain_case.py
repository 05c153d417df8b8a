"""One co-resident TAR+RHT generation on seeded device inputs, saved to .npy:
run in-process (chain kernel) and in a subprocess under OPTR_CHAIN=0 (the
separate pass launches) by test_gpu_parity.test_chain_matches_pass_launches."""

import sys

import numpy as np
import torch

from paper_2310_06993_b200.collectives import MaskSpec, tar_allreduce_local


def run(n: int, L: int, dtype: str, seed: int = 0):
    dev = torch.device("cuda", 0)
    dt = {"f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    g = torch.Generator(device=dev).manual_seed(seed)
    xs = [torch.randn(L, device=dev, generator=g).to(dt) for _ in range(n)]
    outs, counts, got = tar_allreduce_local(xs, rotation=seed % n, ht=True, job_seed=3, generation=seed,
                                            masks=MaskSpec.coin(77 + seed, 0.02), want_received=True)
    torch.cuda.synchronize()
    res = np.stack([o.float().cpu().numpy() for o in outs])
    return res, counts.cpu().numpy(), got.cpu().numpy(), xs


if __name__ == "__main__":
    n, L, dtype, seed, path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4]), sys.argv[5]
    res, counts, got, _ = run(n, L, dtype, seed)
    np.savez(path, res=res, counts=counts, got=got)
