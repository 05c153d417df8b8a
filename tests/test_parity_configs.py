"""Per-element parity at BASELINE.json's configuration shapes (one GPU, the
co-resident n-worker path of ``tar_allreduce_local``) against the oracle.

Every case compares each node's result with the oracle's lossy generation
under the identical masks (north-star bar: RHT on within 1e-5 relative L2
per node; received counts and AllReduceResult.received bit-exact).  The
multi-rank (one worker per process / GPU) counterparts are in
test_multigpu.py.

* the north-star headline bucket, 25,000,000 entries (D = 2^25), 1% coin
  drops, n = 2 and n = 4;
* BASELINE configs[0] exactly: n = 4, 1,048,576 entries, 1% drops;
* the GPT-2 XL bucket (configs[3]): bf16 in, fp32 aggregate, 13,107,200
  entries (D = 2^24), n = 8, 5% coin drops; and the same shape under masks
  captured from the reference's own simulator (SimSession with adaptive
  timeouts, tests/golden/sim_gpt2xl.npz), whose checksums pin the oracle;
* D = 2^26 (the three-pass plan) with 1% drops.
"""

import numpy as np
import pytest

import oracle as O
from golden_util import load

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2310_06993_b200.collectives import MaskSpec, tar_allreduce_local  # noqa: E402

REL = 1e-5


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def _check(dev, buckets, gen, p, coin_seed, seed=9, dtype=torch.float32, spec=None, masks=None,
           want_received=True):
    n, L = len(buckets), len(buckets[0])
    r = gen % n
    dim = O.next_pow2(L)
    if masks is None:
        masks = O.datagram_masks(coin_seed, dim, n, r, p)
    spec = spec or MaskSpec.coin(coin_seed, p)
    xs = [torch.from_numpy(b).to(dev).to(dtype) for b in buckets]
    outs, counts, got = tar_allreduce_local(xs, rotation=r, ht=True, job_seed=seed, generation=gen,
                                            masks=spec, out_dtype=torch.float32, want_received=want_received)
    torch.cuda.synchronize()
    del xs
    res = [o.cpu().numpy() for o in outs]
    gotn = [g.cpu().numpy() for g in got] if got is not None else None
    del outs, got
    c = counts.cpu().numpy()
    inputs = [torch.from_numpy(b).to(dtype).float().numpy() for b in buckets] if dtype != torch.float32 else buckets
    want, _wire, tar = O.run_generation(inputs, seed, gen, True, masks=masks, r=r, return_wire=True, threads=n)
    for node in range(n):
        e = rel_err(res[node], want[node])
        assert e < REL, (node, e)
        if gotn is not None:
            np.testing.assert_array_equal(gotn[node].astype(bool), tar[node][1])
    for (stage, dst), (rcv, _exp) in O.stage_counts(masks, dim, n, r, 350).items():
        assert c[stage - 1, dst] == rcv, (stage, dst)
    return res, want


@pytest.mark.parametrize("n", [2, 4])
def test_headline_25m_one_percent_drops(dev, n):
    buckets = O.make_buckets(31, n, 25_000_000)
    _check(dev, buckets, gen=1, p=0.01, coin_seed=4242, want_received=(n == 2))


def test_cfg1_exact_shape(dev):
    """BASELINE configs[0]: TAR+RHT on one 1M-entry fp32 bucket, 4 workers, 1% drop."""
    buckets = O.make_buckets(0, 4, 1_048_576)
    for gen in range(3):
        _check(dev, buckets, gen=gen, p=0.01, coin_seed=100 + gen)


def test_gpt2xl_bucket_bf16_five_percent(dev):
    """configs[3]: one 25 MB bf16 bucket (13,107,200 entries), n = 8, 5% drops."""
    buckets = O.make_buckets(77, 8, 13_107_200)
    _check(dev, buckets, gen=5, p=0.05, coin_seed=91, dtype=torch.bfloat16, want_received=False)


def test_gpt2xl_bucket_captured_simulator_masks(dev):
    """The GPT-2 XL bucket under the stage-1 / stage-2 masks the reference's
    SimSession consumed (adaptive timeouts + 5% drops), bf16-valued inputs:
    the oracle reproduces the reference's checksums and sampled entries, and
    the GPU matches the oracle per element."""
    z = load("sim_gpt2xl.npz")
    n, L, ht, r, gen_idx, seed, epp, dim = (int(v) for v in z["meta"])
    npk = O.n_packets(dim // n, epp)
    masks = {}
    for dst in range(n):
        for src in range(n):
            if src != dst:
                for stage in (1, 2):
                    bits = np.unpackbits(z[f"m{stage}_{dst}_{src}"], bitorder="little")[:npk]
                    masks[(stage, dst, src)] = bits.astype(bool)
    buckets = [torch.from_numpy(b).to(torch.bfloat16).float().numpy() for b in O.make_buckets(seed, n, L)]
    spec = MaskSpec.from_packets(masks, dim, n, epp * 4, dev)
    res, want = _check(dev, buckets, gen=gen_idx, p=0.0, coin_seed=0, seed=seed, dtype=torch.bfloat16,
                       spec=spec, masks=masks, want_received=False)
    idx = z["sample_idx"]
    for node in range(n):
        # the oracle against the reference's own results (pinned), then the GPU is within 1e-5 of it
        np.testing.assert_allclose(want[node][idx], z["sample_out"][node], rtol=1e-5, atol=1e-6)
        assert abs(want[node].astype(np.float64).sum() - z["out_sum"][node]) < 1e-3 * z["out_norm"][node]
        assert abs(np.linalg.norm(want[node].astype(np.float64)) - z["out_norm"][node]) < 1e-6 * z["out_norm"][node]


def test_three_pass_d26_one_percent_drops(dev):
    """D = 2^26 (three-pass FWHT plan: 32-column strided tiles), n = 2."""
    buckets = O.make_buckets(8, 2, 40_000_000)
    _check(dev, buckets, gen=3, p=0.01, coin_seed=5150, want_received=False)
