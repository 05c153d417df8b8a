"""CPU-side checks of the C ABI: the library loads without a GPU, exports
every symbol include/optr.h declares, and its host ports (SeedSequence,
PCG64 jump-ahead, datagram coin) match numpy / the reference fixtures."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from golden_util import ROOT, load

pkg = pytest.importorskip("paper_2310_06993_b200")
from paper_2310_06993_b200 import _lib  # noqa: E402
from paper_2310_06993_b200.collectives import (  # noqa: E402
    build_schedule, coin_masks_host, expected_counts, owned_shard, pack_packet_masks,
    shard_lengths, shard_offsets, unpack_packet_masks)


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "optr.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(optr_[a-z0-9_]+)\s*\(", txt))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = _header_symbols()
    assert len(syms) >= 19
    assert syms == set(_lib.SIGNATURES), syms ^ set(_lib.SIGNATURES)
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.optr_version()


def test_derive_seed_port_matches_reference_fixture():
    z = load("rng.npz")
    for t, want in zip(z["triples"], z["derive_seed"]):
        assert pkg.derive_seed(*(int(v) for v in t)) == int(want)


def test_pcg64_jump_ahead_matches_reference_fixture():
    z = load("rng.npz")
    lib = _lib.lib()
    for i, s in enumerate(z["raw_seeds"]):
        ent = (ctypes.c_uint64 * 1)(int(s))
        for j, k in enumerate(z["raw_ks"]):
            assert lib.optr_pcg64_output(ent, 1, int(k)) == int(z["raw"][i, j])


def test_pcg64_two_word_entropy_matches_numpy():
    lib = _lib.lib()
    for seed, rank in [(7, 0), (7, 1), (2**40 + 9, 5), (0, 0), (2**64 - 1, 15)]:
        bg = np.random.PCG64(np.random.SeedSequence([seed, rank]))
        want = bg.random_raw(40)
        ent = (ctypes.c_uint64 * 2)(seed, rank)
        got = [lib.optr_pcg64_output(ent, 2, k) for k in range(40)]
        np.testing.assert_array_equal(np.array(got, dtype=np.uint64), want)


@pytest.mark.parametrize("seed,dim,n,r,p,epp", [
    (7, 2048, 2, 0, 0.05, 16), (5, 1000, 3, 2, 0.2, 10), (2**40 + 9, 16384, 4, 3, 0.01, 350),
    (1, 33, 5, 1, 0.3, 2), (3, 7, 8, 0, 0.5, 1), (9, 2**20, 8, 5, 0.01, 350), (4, 100, 4, 1, 0.0, 350)])
def test_host_coin_masks_match_oracle(seed, dim, n, r, p, epp):
    a = coin_masks_host(dim, n, r, seed, p, epp)
    b = O.datagram_masks(seed, dim, n, r, p, epp)
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=str(k))


def test_host_coin_masks_match_live_udp_fixture():
    z = load("datagram.npz")
    for i, run in enumerate(z["runs"]):
        n, ln, rot = int(run[0]), int(run[1]), int(run[2])
        p, seed, mp = float(run[3]), int(run[4]), int(run[5])
        m = coin_masks_host(ln, n, rot, seed, p, mp // 4)
        res = O.tar_masked(list(z[f"in_{i}"]), rot, m, mp // 4)
        for node, (_e, g) in enumerate(res):
            np.testing.assert_array_equal(g, z[f"got_{i}"][node])


def test_packet_mask_pack_roundtrip():
    m = O.datagram_masks(3, 5000, 4, 1, 0.1, 16)
    words = pack_packet_masks(m, 5000, 4, 16)
    back = unpack_packet_masks(words, 5000, 4, 1, 16)
    for k in m:
        np.testing.assert_array_equal(back[k], m[k])


def test_index_helpers_match_oracle():
    for length in [0, 1, 3, 7, 10, 65, 1000, 2**20 + 3]:
        for n in range(2, 9):
            assert shard_lengths(length, n) == O.shard_lengths(length, n)
            assert shard_offsets(length, n) == O.shard_offsets(length, n)
    for n in range(2, 9):
        for r in range(n):
            assert [owned_shard(i, r, n) for i in range(n)] == [O.owned_shard(i, r, n) for i in range(n)]
        for inc in range(1, n):
            sched = build_schedule(n, inc)
            order = [d for rnd in sched.rounds for d in rnd[0]]
            assert order == O.send_order(0, n)


def test_expected_counts_match_oracle():
    for dim, n, r in [(1000, 4, 1), (2**16, 8, 3), (7, 8, 0)]:
        m = O.full_masks(dim, n, r)
        sc = O.stage_counts(m, dim, n, r, 350)
        e = expected_counts(dim, n, r)
        for (stage, dst), (got, exp) in sc.items():
            assert got == exp == e[stage - 1, dst]


def test_invalid_arguments_rejected_without_gpu():
    lib = _lib.lib()
    assert lib.optr_fwht(None, 3, None) == _lib.OPTR_EINVAL
    assert lib.optr_rht_encode(None, 0, 5, None, 4, 0, None) == _lib.OPTR_EINVAL
    assert lib.optr_tar_local_workspace(1, 10, 1, 350) == 0
    assert lib.optr_masks_host(None, 10, 2, 0, 0, 0.1, 350) == _lib.OPTR_EINVAL
    with pytest.raises(ValueError):
        pkg.RhtContext(dim=6, seed=0, orig_len=3)
    with pytest.raises(ValueError):
        pkg.RhtContext(dim=4, seed=0, orig_len=5)


def test_kernel_class_names_match_header():
    """_lib.K_NAMES indexes optr_timing_collect's arrays (optr.h OPTR_K_*)."""
    import re

    from paper_2310_06993_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "optr.h")).read()
    consts = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define OPTR_K_(\w+) (\d+)", hdr)}
    assert consts.pop("CLASSES") == len(_lib.K_NAMES)
    assert sorted(consts.values()) == list(range(len(_lib.K_NAMES)))
