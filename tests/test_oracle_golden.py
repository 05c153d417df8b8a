"""Pin the oracle to golden vectors produced by the real reference.

The fixtures come from tests/golden/make_golden.py (imports ubar from
/root/reference).  These tests need no GPU and no reference checkout.
"""

import os

import numpy as np
import pytest

import oracle as O
from golden_util import GOLDEN, load


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def test_derive_seed_matches_reference():
    z = _load("rng.npz")
    for t, want in zip(z["triples"], z["derive_seed"]):
        assert O.derive_seed(*(int(v) for v in t)) == int(want)


def test_signs_match_reference():
    z = _load("rng.npz")
    for dim, seed in z["sign_cases"]:
        dim, seed = int(dim), int(seed)
        bits = np.packbits(O.rht_signs(dim, seed) > 0, bitorder="little")
        np.testing.assert_array_equal(bits, z[f"signs_{dim}_{seed}"])


def test_coin_stream_matches_reference():
    z = _load("rng.npz")
    for (s, r), want in zip(z["coin_keys"], z["coins"]):
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(s), int(r)])))
        np.testing.assert_array_equal(g.random(64), want)


def test_codec_matches_reference():
    z = _load("codec.npz")
    for ln in z["lengths"]:
        ln = int(ln)
        seed = int(z[f"seed_{ln}"])
        dim = O.next_pow2(ln)
        signs = O.rht_signs(dim, seed)
        y = O.rht_encode(z[f"x_{ln}"], dim, signs)
        np.testing.assert_array_equal(y, z[f"y_{ln}"])
        keep = z[f"keep_{ln}"]
        dec = O.rht_decode(np.where(keep, y, 0.0), keep, ln, signs)
        np.testing.assert_array_equal(dec, z[f"dec_{ln}"])
        full = O.rht_decode(y, np.ones(dim, bool), ln, signs)
        np.testing.assert_array_equal(full, z[f"full_{ln}"])


def test_lossless_tar_matches_reference():
    z = _load("lossless.npz")
    for idx, (n, ln, r, _incast) in enumerate(z["cases"]):
        buckets = list(z[f"in_{idx}"])
        res = O.tar_masked(buckets, int(r), O.full_masks(int(ln), int(n), int(r)), 350)
        for node, (e, g) in enumerate(res):
            np.testing.assert_array_equal(e, z[f"out_{idx}"][node])
            np.testing.assert_array_equal(g, z[f"got_{idx}"][node])


def test_datagram_coin_masks_match_live_udp_runs():
    """Counter-indexed coin model == what live loopback UDP runs consumed;
    the HT-off TAR result is bit-exact."""
    z = _load("datagram.npz")
    for i, run in enumerate(z["runs"]):
        n, ln, rot = int(run[0]), int(run[1]), int(run[2])
        p, seed, mp = float(run[3]), int(run[4]), int(run[5])
        masks = O.datagram_masks(seed, ln, n, rot, p, epp=mp // 4)
        res = O.tar_masked(list(z[f"in_{i}"]), rot, masks, mp // 4)
        for node, (e, g) in enumerate(res):
            np.testing.assert_array_equal(g, z[f"got_{i}"][node])
            np.testing.assert_array_equal(e, z[f"out_{i}"][node])


def _sim_masks(z, key, n):
    m = {}
    for dst in range(n):
        for src in range(n):
            if src != dst:
                m[(1, dst, src)] = z[f"{key}_m1_{dst}_{src}"]
                m[(2, dst, src)] = z[f"{key}_m2_{dst}_{src}"]
    return m


def test_sim_replay_matches_reference_generation():
    """Captured simulator masks replayed through the oracle reproduce
    SimSession.run_generation bit-for-bit (HT on and off)."""
    z = _load("sim.npz")
    for ci, gens in enumerate(z["gens"]):
        for g in range(int(gens)):
            key = f"c{ci}_g{g}"
            n, L, ht, r, gen_idx, seed, epp, dim = (int(v) for v in z[f"{key}_meta"])
            masks = _sim_masks(z, key, n)
            out = O.run_generation(list(z[f"{key}_in"]), seed, gen_idx, bool(ht),
                                   masks=masks, r=r, epp=epp)
            for node in range(n):
                np.testing.assert_array_equal(out[node], z[f"{key}_out"][node])


def test_shard_and_owner_pins():
    # test_wire.py:111-118, test_schedule.py:14-25
    assert O.shard_lengths(10, 4) == [3, 3, 2, 2]
    assert O.shard_lengths(3, 4) == [1, 1, 1, 0]
    assert O.shard_offsets(10, 4) == [0, 3, 6, 8, 10]
    for n in range(2, 9):
        for r in range(n):
            for j in range(n):
                assert O.owned_shard(O.shard_owner(j, r, n), r, n) == j


def test_fwht_dense_sylvester():
    import scipy.linalg
    for d in [1, 2, 4, 8, 64, 128]:
        h = scipy.linalg.hadamard(d).astype(np.float64) if d > 1 else np.ones((1, 1))
        x = np.random.default_rng(d).standard_normal(d)
        np.testing.assert_allclose(O.fwht(x.copy()), h @ x, rtol=1e-10, atol=1e-10)
    with pytest.raises(ValueError):
        O.fwht(np.zeros(3))


def _bf16(x):
    """float32 -> bfloat16 (ties to even) as float32, like make_golden.bf16_round."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def test_sim_capture_gpt2xl_shape_replays_reference():
    """The reference's SimSession at the GPT-2 XL bucket shape (n=8,
    13,107,200 bf16-valued entries, 5% drops, adaptive timeouts; masks
    captured at consumption time) is reproduced exactly by the oracle:
    sampled entries bit-equal, per-node sums equal."""
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
    lost = sum(int((~m).sum()) for m in masks.values()) / sum(len(m) for m in masks.values())
    assert 0.0 < lost <= 0.06  # configs[3]: adaptive-timeout masks up to ~5%
    want = O.run_generation([_bf16(b) for b in O.make_buckets(seed, n, L)], seed, gen_idx, bool(ht),
                            masks=masks, r=r, epp=epp, threads=n)
    idx = z["sample_idx"]
    for node in range(n):
        np.testing.assert_array_equal(want[node][idx], z["sample_out"][node])
        assert want[node].astype(np.float64).sum() == z["out_sum"][node]
