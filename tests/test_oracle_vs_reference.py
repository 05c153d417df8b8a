"""Oracle vs the live reference (build container only: needs /root/reference).

Randomised SimSession generations (lossy UBT, adaptive timeouts, HT on/off)
are run by the real `ubar`, their consumed masks captured at consumption
time, and replayed through the oracle: results must be bit-identical.  The
datagram coin model and the codec are checked the same way.
"""

import os
import sys

import numpy as np
import pytest

import oracle as O

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.reference

if not os.path.isdir(REF):
    pytest.skip("reference checkout not present", allow_module_level=True)

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
sys.dont_write_bytecode = True
import make_golden as MG  # noqa: E402  (imports ubar from /root/reference)

import ubar.collectives as ucoll  # noqa: E402
from ubar.config import ExperimentConfig  # noqa: E402
from ubar.hadamard import DropMask, RhtContext, derive_seed, rht_decode, rht_encode  # noqa: E402
from ubar.harness import _bucket_rng, build_session  # noqa: E402
from ubar.schedule import owned_shard  # noqa: E402
from ubar.wire import shard_offsets  # noqa: E402


@pytest.mark.parametrize("case", range(6))
def test_sim_generations_replay_bit_exact(case):
    rng = np.random.default_rng(900 + case)
    n = int(rng.integers(2, 9))
    L = int(rng.integers(500, 20000))
    ht = "on" if case % 2 == 0 else "off"
    p = float(rng.choice([0.01, 0.03, 0.08]))
    cfg = ExperimentConfig(n=n, bucket_len=L, ht=ht, drop_prob=p, p99_over_p50=float(rng.choice([1.5, 3.0])),
                           latency_distribution=str(rng.choice(["mixture", "lognormal"])), seed=case,
                           calibration_iterations=3)
    session = build_session(cfg)
    brng = _bucket_rng(cfg)
    epp = cfg.max_payload // 4
    for _g in range(2):
        buckets = [brng.standard_normal(L).astype(np.float32) for _ in range(n)]
        log, orig = MG._capture_stage1()
        try:
            r, gen = session.rotation, session.generation
            report = session.run_generation(buckets)
        finally:
            ucoll._mean_received = orig
        log = log[-n:]
        dim = len(report.stats[0].result.entries)
        offs = shard_offsets(dim, n)
        masks = {}
        for rank, mk in log:
            for src, m in mk.items():
                masks[(1, rank, src)] = MG._to_packets(m, epp)
        for dst, st in enumerate(report.stats):
            got = np.asarray(st.result.received)
            for src in range(n):
                if src != dst:
                    j = owned_shard(src, r, n)
                    masks[(2, dst, src)] = MG._to_packets(got[offs[j]:offs[j + 1]], epp)
        out = O.run_generation(buckets, case, gen, ht == "on", masks=masks, r=r, epp=epp)
        for node in range(n):
            np.testing.assert_array_equal(out[node], report.results[node])


def test_codec_against_reference_random():
    rng = np.random.default_rng(5)
    for _ in range(30):
        ln = int(rng.integers(1, 5000))
        seed = derive_seed(int(rng.integers(0, 2**40)), int(rng.integers(0, 65536)), int(rng.integers(0, 2**20)))
        ctx = RhtContext.for_length(ln, seed)
        np.testing.assert_array_equal(O.rht_signs(ctx.dim, seed), ctx.signs)
        x = rng.standard_normal(ln)
        y = rht_encode(x, ctx)
        np.testing.assert_array_equal(O.rht_encode(x, ctx.dim, ctx.signs), y)
        keep = rng.random(ctx.dim) >= 0.2
        keep[0] = True
        np.testing.assert_array_equal(O.rht_decode(np.where(keep, y, 0.0), keep, ln, ctx.signs),
                                      rht_decode(np.where(keep, y, 0.0), DropMask(keep), ctx))
