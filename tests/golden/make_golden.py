"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``ubar`` read-only from /root/reference/pkg/src and records what the
reference itself produces on fixed seeds:

* ``rng.npz``      -- derive_seed values, PCG64 raw outputs at chosen indices,
                      Rademacher sign bits, ``random()`` coin streams
                      (hadamard.py:31-51, datagram.py:70-72,122).
* ``codec.npz``    -- rht_encode / rht_decode vectors over awkward lengths and
                      a random drop mask (hadamard.py:93-123).
* ``lossless.npz`` -- tar_allreduce driven by run_lossless over n, rotation,
                      incast and awkward lengths (collectives.py:97-150,321).
* ``datagram.npz`` -- live loopback UDP TAR runs with the seeded send-side
                      coin: per-node entries + received (datagram.py:85-207).
* ``sim.npz``      -- SimSession.run_generation with lossy UBT + adaptive
                      timeouts; the consumed stage-1/stage-2 masks are
                      captured at consumption time (SURVEY finding 2/5) and
                      stored per packet, next to the reference results
                      (runner.py:211-276).
* ``wire.npz``     -- packet byte streams of wire.iter_packets + encode_header
                      (wire.py:36-85,183-208) over awkward shard lengths,
                      header fields and payload sizes.
* ``sim_gpt2xl.npz`` -- the same capture at the GPT-2 XL bucket shape
                      (BASELINE configs[3]: n=8, 13,107,200 entries, bf16-valued
                      inputs, 5% drops, adaptive timeouts): packed packet masks
                      plus per-node checksums and sampled entries of the
                      reference's results (the full outputs are 420 MB).

Nothing here runs on the GPU box; the .npz files travel instead.
"""

from __future__ import annotations

import socket
import sys
import threading
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import ubar.collectives as ucoll  # noqa: E402
from ubar.collectives import run_lossless, tar_allreduce  # noqa: E402
from ubar.datagram import DatagramEndpoint  # noqa: E402
from ubar.hadamard import DropMask, RhtContext, derive_seed, rht_decode, rht_encode  # noqa: E402
from ubar.harness import _bucket_rng, build_session  # noqa: E402
from ubar.config import ExperimentConfig  # noqa: E402
from ubar.schedule import Topology, build_schedule, owned_shard  # noqa: E402
from ubar.wire import shard_offsets  # noqa: E402

OUT = Path(__file__).resolve().parent


def pack_pm1(signs: np.ndarray) -> np.ndarray:
    return np.packbits(signs > 0, bitorder="little")


def gen_rng():
    triples = np.array(
        [(0, 0, 0), (1, 2, 3), (1, 2, 4), (1, 3, 3), (2, 2, 3), (7, 7, 7),
         (0, 1, 1), (0, 65535, 65535), (0, 0, 65536), (123456789, 42, 99999),
         (2**32 + 5, 3, 2**33 + 1), (2**64 - 1, 0, 1)],
        dtype=object,
    )
    seeds = np.array([int(derive_seed(*t)) for t in triples], dtype=np.uint64)

    # raw PCG64 outputs out(k) at chosen k, for several u64 seeds
    raw_seeds = [0, 1, 99, 2**32 + 1, int(seeds[1]), 2**64 - 1]
    ks = np.array([0, 1, 2, 3, 7, 31, 32, 1000, 123457, (1 << 24) + 5, (1 << 40) + 3],
                  dtype=np.uint64)
    raw = np.zeros((len(raw_seeds), len(ks)), dtype=np.uint64)
    for i, s in enumerate(raw_seeds):
        for jj, k in enumerate(ks):
            bg = np.random.PCG64(np.random.SeedSequence(s))
            bg.advance(int(k))
            raw[i, jj] = bg.random_raw()

    # Rademacher signs exactly as RhtContext builds them
    sign_cases = [(2, 99), (16, 0), (64, 10), (1024, 5), (4096, 123), (1 << 16, int(seeds[0])),
                  (1 << 20, derive_seed(0, 0, 0))]
    sign_bits = {}
    for dim, s in sign_cases:
        sign_bits[f"signs_{dim}_{s}"] = pack_pm1(RhtContext(dim=dim, seed=s, orig_len=dim).signs)

    # datagram coin stream: PCG64(SeedSequence([seed, rank])).random()
    coin_keys = [(7, 0), (7, 1), (0, 3), (2**40 + 9, 5)]
    coins = np.zeros((len(coin_keys), 64))
    for i, (s, r) in enumerate(coin_keys):
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([s, r])))
        coins[i] = g.random(64)

    np.savez_compressed(
        OUT / "rng.npz",
        triples=np.array([[int(v) for v in t] for t in triples], dtype=object).astype(str),
        derive_seed=seeds,
        raw_seeds=np.array([str(s) for s in raw_seeds]),
        raw_ks=ks,
        raw=raw,
        sign_cases=np.array([(d, str(s)) for d, s in sign_cases], dtype=object).astype(str),
        coin_keys=np.array([(str(s), r) for s, r in coin_keys], dtype=object).astype(str),
        coins=coins,
        **sign_bits,
    )


def gen_codec():
    lengths = [1, 2, 3, 5, 8, 17, 100, 333, 1000, 2048, 4095, 4096, 5000]
    rng = np.random.default_rng(2310)
    rec = {}
    for ln in lengths:
        seed = derive_seed(11, ln % 65536, ln)
        ctx = RhtContext.for_length(ln, seed)
        x = rng.standard_normal(ln).astype(np.float32)
        y = rht_encode(x, ctx)
        keep = rng.random(ctx.dim) >= 0.1
        if not keep.any():
            keep[0] = True
        dec = rht_decode(np.where(keep, y, 0.0), DropMask(keep), ctx)
        full = rht_decode(y, DropMask.full(ctx.dim), ctx)
        rec[f"x_{ln}"] = x
        rec[f"seed_{ln}"] = np.array(str(seed))
        rec[f"y_{ln}"] = y
        rec[f"keep_{ln}"] = keep
        rec[f"dec_{ln}"] = dec
        rec[f"full_{ln}"] = full
    np.savez_compressed(OUT / "codec.npz", lengths=np.array(lengths), **rec)


def gen_lossless():
    cases = []
    rec = {}
    idx = 0
    for n, ln, r, incast in [(2, 1000, 0, 1), (3, 1000, 2, 2), (4, 7, 1, 1), (4, 65, 3, 3),
                             (5, 1000, 4, 1), (6, 97, 5, 5), (8, 1000, 3, 1), (8, 3, 0, 7),
                             (4, 1, 2, 1)]:
        rng = np.random.default_rng(idx + 77)
        buckets = [rng.standard_normal(ln).astype(np.float32) for _ in range(n)]
        if idx == 6:  # collectives test 99-108: 1e6 offset, fp64 accumulation
            buckets = [(1e6 + rng.standard_normal(ln)).astype(np.float32) for _ in range(n)]
        gens = [tar_allreduce(i, buckets[i], Topology(n), r, build_schedule(n, incast))
                for i in range(n)]
        res = run_lossless(gens)
        rec[f"in_{idx}"] = np.stack(buckets)
        rec[f"out_{idx}"] = np.stack([x.entries for x in res])
        rec[f"got_{idx}"] = np.stack([x.received for x in res])
        cases.append((n, ln, r, incast))
        idx += 1
    np.savez_compressed(OUT / "lossless.npz", cases=np.array(cases), **rec)


def _free_ports(k):
    socks = [socket.socket(socket.AF_INET, socket.SOCK_DGRAM) for _ in range(k)]
    for s in socks:
        s.bind(("127.0.0.1", 0))
    ports = [s.getsockname()[1] for s in socks]
    for s in socks:
        s.close()
    return ports


def _udp_group(n, buckets, rotation, drop_prob, seed, max_payload, t_b=2.0):
    ports = _free_ports(n)
    addrs = {r: ("127.0.0.1", ports[r]) for r in range(n)}
    eps = [DatagramEndpoint(r, addrs, t_b=t_b, drop_prob=drop_prob, seed=seed,
                            max_payload=max_payload) for r in range(n)]
    sched = build_schedule(n, incast=n - 1)
    results = [None] * n
    errs = []

    def worker(r):
        try:
            results[r] = eps[r].run(tar_allreduce(r, buckets[r], Topology(n), rotation, sched))
        except Exception as exc:  # pragma: no cover
            errs.append(exc)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    for ep in eps:
        ep.close()
    if errs:
        raise errs[0]
    return results


def gen_datagram():
    """Live loopback runs (test_datagram.py:26-54 harness).  The per-rank
    ``received`` flags are exactly the consumed masks."""
    runs = [
        # n, length, rotation, drop, seed, max_payload
        (2, 2048, 0, 0.05, 7, 64),
        (4, 333, 2, 0.10, 3, 64),
        (4, 4096, 1, 0.05, 12, 1400),
        (3, 1000, 2, 0.2, 5, 40),
        (4, 16384, 3, 0.01, 2**40 + 9, 1400),
    ]
    rec = {}
    for i, (n, ln, rot, p, seed, mp) in enumerate(runs):
        rng = np.random.default_rng(500 + i)
        buckets = [rng.standard_normal(ln).astype(np.float32) for _ in range(n)]
        # The live backend also cuts stages on wall-clock timeouts, and with
        # a coin-dropped last-percentile packet two hard timeouts of equal
        # t_B can race (datagram.py:165-191).  Keep a run only when three
        # live repetitions agree exactly, so the fixture records the
        # deterministic (coin) behaviour, not a lost race.
        def agree(reps):
            return all(np.array_equal(np.asarray(a.received), np.asarray(b.received))
                       for rep in reps[1:] for a, b in zip(reps[0], rep))

        for attempt in range(20):
            reps = [_udp_group(n, buckets, rot, p, seed, mp) for _ in range(3)]
            if agree(reps):
                break
            seed += 1000  # lost a timeout race: move to another coin seed
        else:
            raise RuntimeError(f"run {i}: no race-free seed found")
        runs[i] = (n, ln, rot, p, seed, mp)
        res = reps[0]
        rec[f"in_{i}"] = np.stack(buckets)
        rec[f"out_{i}"] = np.stack([np.asarray(x.entries) for x in res])
        rec[f"got_{i}"] = np.stack([np.asarray(x.received) for x in res])
    np.savez_compressed(OUT / "datagram.npz",
                        runs=np.array([[str(v) for v in r] for r in runs]), **rec)


def _capture_stage1():
    """Wrap collectives._mean_received to copy each owner's consumed stage-1
    masks at call time (the live dicts keep changing, simdriver.py:342)."""
    log = []
    orig = ucoll._mean_received

    def shim(rank, own, result, n):
        log.append((rank, {p: np.array(m, copy=True) for p, m in result.mask.items()}))
        return orig(rank, own, result, n)

    ucoll._mean_received = shim
    return log, orig


def _to_packets(mask: np.ndarray, epp: int) -> np.ndarray:
    npk = -(-len(mask) // epp) if len(mask) else 0
    pk = np.zeros(npk, bool)
    for k in range(npk):
        seg = mask[k * epp:(k + 1) * epp]
        assert seg.all() or not seg.any(), "mask not packet-uniform"
        pk[k] = bool(seg[0])
    return pk


def gen_sim():
    configs = [
        # n, L, ht, drop, p99/50, dist, gens, seed
        (4, 16384, "on", 0.01, 3.0, "lognormal", 3, 1),
        (8, 10000, "on", 0.05, 1.5, "mixture", 2, 2),
        (4, 12345, "off", 0.02, 3.0, "lognormal", 2, 3),
    ]
    rec = {}
    for ci, (n, L, ht, p, ratio, dist, gens, seed) in enumerate(configs):
        cfg = ExperimentConfig(n=n, bucket_len=L, ht=ht, drop_prob=p, p99_over_p50=ratio,
                               latency_distribution=dist, seed=seed, generations=gens,
                               calibration_iterations=5)
        session = build_session(cfg)
        brng = _bucket_rng(cfg)
        epp = cfg.max_payload // 4
        for g in range(gens):
            buckets = [brng.standard_normal(L).astype(np.float32) for _ in range(n)]
            log, orig = _capture_stage1()
            try:
                r = session.rotation
                gen_idx = session.generation
                report = session.run_generation(buckets)
            finally:
                ucoll._mean_received = orig
            dim = len(report.stats[0].result.entries)
            offs = shard_offsets(dim, n)
            log = log[-n:]  # earlier calls were the calibration runs (runner.py:138-187)
            assert len(log) == n
            key = f"c{ci}_g{g}"
            pk1 = {}
            for rank, masks in log:
                for src, m in masks.items():
                    pk1[(rank, src)] = _to_packets(m, epp)
            pk2 = {}
            for dst, st in enumerate(report.stats):
                got = np.asarray(st.result.received)
                for src in range(n):
                    if src == dst:
                        continue
                    j = owned_shard(src, r, n)
                    pk2[(dst, src)] = _to_packets(got[offs[j]:offs[j + 1]], epp)
            for (dst, src), v in pk1.items():
                rec[f"{key}_m1_{dst}_{src}"] = v
            for (dst, src), v in pk2.items():
                rec[f"{key}_m2_{dst}_{src}"] = v
            rec[f"{key}_in"] = np.stack(buckets)
            rec[f"{key}_out"] = np.stack([np.asarray(x) for x in report.results])
            rec[f"{key}_meta"] = np.array([n, L, int(report.ht_used), r, gen_idx, seed, epp, dim])
            rec[f"{key}_loss"] = np.array([s.loss_rate for s in report.stats])
    np.savez_compressed(OUT / "sim.npz",
                        configs=np.array([[str(v) for v in c] for c in configs]),
                        gens=np.array([c[6] for c in configs]), **rec)


def gen_wire():
    from ubar.wire import encode_header, iter_packets

    cases = [
        # entries, bucket_id, base_offset, max_payload, timeout_share, incast
        (0, 1, 0, 1400, 0, 0), (1, 2, 0, 1400, 0, 0), (349, 7, 4, 1400, 3, 1), (350, 65535, 0, 1400, 255, 127),
        (351, 0, 1400, 1400, 17, 5), (1000, 300, 12, 64, 9, 0), (35_000, 42, 0, 1400, 128, 3),
        (100_001, 9, 4_000_000, 1400, 1, 2),
    ]
    rec = {}
    for i, (ne, bid, base, mp, ts, inc) in enumerate(cases):
        x = np.random.default_rng(700 + i).standard_normal(ne).astype(np.float32)
        pk = [encode_header(h) + p for h, p in iter_packets(bid, x.tobytes(), base, mp, ts, inc)]
        rec[f"x_{i}"] = x
        rec[f"lens_{i}"] = np.array([len(p) for p in pk], dtype=np.int64)
        rec[f"bytes_{i}"] = np.frombuffer(b"".join(pk), dtype=np.uint8)
    np.savez_compressed(OUT / "wire.npz", cases=np.array(cases, dtype=np.int64), **rec)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bfloat16 (ties to even), kept as float32 (torch's
    .to(torch.bfloat16) on finite values)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def gen_sim_large():
    n, L, p, ratio, dist, seed = 8, 13_107_200, 0.05, 3.0, "lognormal", 5
    cfg = ExperimentConfig(n=n, bucket_len=L, ht="on", drop_prob=p, p99_over_p50=ratio,
                           latency_distribution=dist, seed=seed, calibration_iterations=3)
    session = build_session(cfg)
    brng = _bucket_rng(cfg)
    epp = cfg.max_payload // 4
    buckets = [bf16_round(brng.standard_normal(L).astype(np.float32)) for _ in range(n)]
    log, orig = _capture_stage1()
    try:
        r = session.rotation
        gen_idx = session.generation
        report = session.run_generation(buckets)
    finally:
        ucoll._mean_received = orig
    dim = len(report.stats[0].result.entries)
    offs = shard_offsets(dim, n)
    log = log[-n:]
    rec = {}
    for rank, masks in log:
        for src, m in masks.items():
            rec[f"m1_{rank}_{src}"] = np.packbits(_to_packets(m, epp), bitorder="little")
    for dst, st in enumerate(report.stats):
        got = np.asarray(st.result.received)
        for src in range(n):
            if src != dst:
                j = owned_shard(src, r, n)
                rec[f"m2_{dst}_{src}"] = np.packbits(_to_packets(got[offs[j]:offs[j + 1]], epp), bitorder="little")
    outs = np.stack([np.asarray(x, dtype=np.float32) for x in report.results])
    idx = np.random.default_rng(0).choice(L, 4096, replace=False)
    rec["sample_idx"] = idx
    rec["sample_out"] = outs[:, idx]
    rec["out_sum"] = outs.astype(np.float64).sum(axis=1)
    rec["out_norm"] = np.linalg.norm(outs.astype(np.float64), axis=1)
    rec["meta"] = np.array([n, L, int(report.ht_used), r, gen_idx, seed, epp, dim])
    rec["loss"] = np.array([s.loss_rate for s in report.stats])
    np.savez_compressed(OUT / "sim_gpt2xl.npz", **rec)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "codec", "lossless", "datagram", "sim", "sim_large", "wire"]
    for w in which:
        globals()[f"gen_{w}"]()
        print("wrote", w)
