"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference hot path.

Not product code: see ``oracle/__init__.py`` for who may import this.
Citations are ``file:line`` into ``/root/reference/pkg/src/ubar/``.

Mask convention shared with the product:
a mask set maps ``(stage, dst, src) -> bool[n_packets]`` where packet ``k`` of
the shard ``src`` sends to ``dst`` in ``stage`` covers entries
``[k*epp, min((k+1)*epp, len))``.  Stage 1 carries shard
``owned_shard(dst, r, n)`` (collectives.py:117-122), stage 2 carries shard
``owned_shard(src, r, n)`` (collectives.py:133-137).  Every packet of every
simulator / datagram run is all-or-nothing (simdriver.py:186-190,258-272;
datagram.py:117-124,150-159), so packet granularity loses nothing.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "ENTRY_BYTES",
    "MAX_PAYLOAD",
    "EmptyReception",
    "next_pow2",
    "derive_seed",
    "rht_signs",
    "fwht",
    "rht_encode",
    "rht_decode",
    "shard_lengths",
    "shard_offsets",
    "owned_shard",
    "shard_owner",
    "send_order",
    "n_packets",
    "datagram_masks",
    "full_masks",
    "expand_packets",
    "mean_received",
    "tar_masked",
    "run_generation",
    "bucket_rng",
    "make_buckets",
    "oracle_allreduce",
    "stage_counts",
]

ENTRY_BYTES = 4  # wire.py:23
MAX_PAYLOAD = 1400  # wire.py:22


class EmptyReception(RuntimeError):
    """hadamard.py:17-18 EmptyReceptionError."""


# --------------------------------------------------------------------------
# codec  (hadamard.py)
# --------------------------------------------------------------------------


def next_pow2(n: int) -> int:
    """hadamard.py:25-28."""
    if n <= 1:
        return 1
    return 1 << (int(n) - 1).bit_length()


def derive_seed(job_seed: int, bucket_id: int, generation: int) -> int:
    """hadamard.py:31-34 (runner passes bucket_id = generation % 65536,
    runner.py:219-222)."""
    ss = np.random.SeedSequence([int(job_seed), int(bucket_id), int(generation)])
    return int(ss.generate_state(1, dtype=np.uint64)[0])


def rht_signs(dim: int, seed: int) -> np.ndarray:
    """hadamard.py:49-51: Rademacher diagonal as float64 +-1."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence(int(seed))))
    return rng.integers(0, 2, size=dim).astype(np.float64) * 2.0 - 1.0


def fwht(v: np.ndarray) -> np.ndarray:
    """hadamard.py:76-90: unnormalised Sylvester (natural order) WHT, in place
    on a contiguous copy's view; returns the transformed array."""
    v = np.ascontiguousarray(v)
    d = len(v)
    if d <= 0 or (d & (d - 1)) != 0:
        raise ValueError(f"length must be a power of two, got {d}")
    h = 1
    while h < d:
        blocks = v.reshape(-1, 2 * h)
        a = blocks[:, :h].copy()
        b = blocks[:, h:]
        blocks[:, :h] = a + b
        blocks[:, h:] = a - b
        h *= 2
    return v


def rht_encode(x: np.ndarray, dim: int, signs: np.ndarray) -> np.ndarray:
    """hadamard.py:93-102: y = H (signs * pad(x)) / sqrt(dim), float64."""
    x = np.asarray(x, dtype=np.float64)
    padded = np.zeros(dim, dtype=np.float64)
    padded[: len(x)] = x
    y = fwht(padded * signs)
    y /= np.sqrt(dim)
    return y


def rht_decode(y_recv: np.ndarray, received: np.ndarray, orig_len: int,
               signs: np.ndarray) -> np.ndarray:
    """hadamard.py:105-123: global scale dim/count(received), zero-fill misses,
    x = signs * H(y) / sqrt(dim), truncated to orig_len.  float64."""
    y_recv = np.asarray(y_recv, dtype=np.float64)
    dim = len(y_recv)
    cnt = int(np.asarray(received, dtype=bool).sum())
    if cnt == 0:
        raise EmptyReception("no transformed entries received")
    scale = dim / cnt
    y = np.where(received, y_recv, 0.0) * scale
    x = signs * fwht(y)
    x /= np.sqrt(dim)
    return x[:orig_len]


# --------------------------------------------------------------------------
# sharding / ownership / schedule  (wire.py, schedule.py)
# --------------------------------------------------------------------------


def shard_lengths(length: int, n: int) -> list[int]:
    """wire.py:121-126: ceiling split, the first length%n shards get +1."""
    base, extra = divmod(int(length), n)
    return [base + 1 if j < extra else base for j in range(n)]


def shard_offsets(length: int, n: int) -> list[int]:
    """wire.py:129-133: n+1 fence posts."""
    offs = [0]
    for ln in shard_lengths(length, n):
        offs.append(offs[-1] + ln)
    return offs


def shard_owner(j: int, r: int, n: int) -> int:
    """schedule.py:42-44."""
    return (j + r) % n


def owned_shard(node: int, r: int, n: int) -> int:
    """schedule.py:47-49."""
    return (node - r) % n


def send_order(src: int, n: int) -> list[int]:
    """schedule.py:67-78 concatenated over rounds: offsets 1..n-1 in order,
    independent of the incast factor I."""
    return [(src + o) % n for o in range(1, n)]


def n_packets(n_entries: int, epp: int) -> int:
    """wire.py:176-180 / simdriver.py:186-189: ceil(entries / epp), 0 for 0."""
    return -(-int(n_entries) // epp) if n_entries > 0 else 0


# --------------------------------------------------------------------------
# drop masks
# --------------------------------------------------------------------------


def full_masks(dim: int, n: int, r: int, epp: int = MAX_PAYLOAD // ENTRY_BYTES) -> dict:
    """Lossless channel (collectives.py:321-401): every packet delivered."""
    lens = shard_lengths(dim, n)
    out = {}
    for dst in range(n):
        for src in range(n):
            if src == dst:
                continue
            out[(1, dst, src)] = np.ones(n_packets(lens[owned_shard(dst, r, n)], epp), bool)
            out[(2, dst, src)] = np.ones(n_packets(lens[owned_shard(src, r, n)], epp), bool)
    return out


def datagram_masks(seed: int, dim: int, n: int, r: int, drop_prob: float,
                   epp: int = MAX_PAYLOAD // ENTRY_BYTES) -> dict:
    """Send-side seeded drop coin of the UDP backend.

    datagram.py:70-72: sender ``src`` owns ``PCG64(SeedSequence([seed, src]))``;
    datagram.py:117-124: one ``rng.random()`` per packet, in send order, drop
    iff ``< drop_prob`` (no draw at all when drop_prob == 0);
    collectives.py:117-122 / 133-137: stage 1 then stage 2, destinations in
    schedule order (schedule.py:67-78).
    """
    lens = shard_lengths(dim, n)
    out = {}
    for src in range(n):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), src])))
        for stage in (1, 2):
            for dst in send_order(src, n):
                j = owned_shard(dst, r, n) if stage == 1 else owned_shard(src, r, n)
                npk = n_packets(lens[j], epp)
                if drop_prob > 0:
                    coins = rng.random(npk)
                    out[(stage, dst, src)] = ~(coins < drop_prob)
                else:
                    out[(stage, dst, src)] = np.ones(npk, bool)
    return out


def expand_packets(pk: np.ndarray, length: int, epp: int) -> np.ndarray:
    """Packet flags -> per-entry flags over a shard of ``length`` entries."""
    return np.repeat(np.asarray(pk, bool), epp)[:length]


def stage_counts(masks: dict, dim: int, n: int, r: int, epp: int) -> dict:
    """Per (stage, dst): (received_entries, expected_entries) -- the numbers
    StageOutcome carries as bytes/4 (simdriver.py:328-341)."""
    lens = shard_lengths(dim, n)
    out = {}
    for (stage, dst, src), pk in masks.items():
        j = owned_shard(dst, r, n) if stage == 1 else owned_shard(src, r, n)
        e = expand_packets(pk, lens[j], epp)
        got, exp = out.get((stage, dst), (0, 0))
        out[(stage, dst)] = (got + int(e.sum()), exp + lens[j])
    return out


# --------------------------------------------------------------------------
# TAR  (collectives.py)
# --------------------------------------------------------------------------


def mean_received(rank: int, own: np.ndarray, data: dict, mask: dict, n: int) -> np.ndarray:
    """collectives.py:77-94: float64 accumulate in ascending node order, own
    shard counted once, peers add (zero-filled) data and their mask; divide
    where count>0 else 0; cast float32."""
    acc = np.zeros(len(own), dtype=np.float64)
    cnt = np.zeros(len(own), dtype=np.float64)
    for i in range(n):
        if i == rank:
            acc += own
            cnt += 1.0
        elif i in data:
            acc += data[i]
            cnt += mask[i]
    out = np.divide(acc, cnt, out=np.zeros_like(acc), where=cnt > 0)
    return out.astype(np.float32)


def tar_masked(wire: list, r: int, masks: dict, epp: int, entry_masks: dict | None = None) -> list:
    """collectives.py:97-150 over a channel that delivers exactly the packets
    ``masks`` marks (zero-filled misses, simdriver.py:245-247,270-271).

    ``wire``: n float32 vectors of equal length.  Returns per node
    ``(entries float32, received bool)`` (AllReduceResult, :65-74).
    ``entry_masks``: optional {(stage, dst, src): bool[shard len]} replacing
    the packet expansion (e.g. a stage-1 deadline cut mid-packet).
    """
    entry_masks = entry_masks or {}

    def emask(key, ln):
        return entry_masks[key] if key in entry_masks else expand_packets(masks[key], ln, epp)

    n = len(wire)
    wire = [np.asarray(w, dtype=np.float32) for w in wire]
    length = len(wire[0])
    offs = shard_offsets(length, n)

    def shard(node, j):
        return wire[node][offs[j]:offs[j + 1]]

    # stage 1: owner `dst` receives shard my_j from every peer (:113-125)
    s_r = {}
    for dst in range(n):
        j = owned_shard(dst, r, n)
        ln = offs[j + 1] - offs[j]
        data, mk = {}, {}
        for src in range(n):
            if src == dst:
                continue
            e = emask((1, dst, src), ln)
            data[src] = np.where(e, shard(src, j), np.float32(0.0)).astype(np.float32)
            mk[src] = e
        s_r[dst] = mean_received(dst, shard(dst, j).astype(np.float64), data, mk, n)

    # stage 2: every node receives each peer's aggregated shard (:127-150)
    results = []
    for dst in range(n):
        out = np.zeros(length, dtype=np.float32)
        got = np.zeros(length, dtype=bool)
        my_j = owned_shard(dst, r, n)
        out[offs[my_j]:offs[my_j + 1]] = s_r[dst]
        got[offs[my_j]:offs[my_j + 1]] = True
        for src in range(n):
            if src == dst:
                continue
            j = owned_shard(src, r, n)
            ln = offs[j + 1] - offs[j]
            e = emask((2, dst, src), ln)
            out[offs[j]:offs[j + 1]] = np.where(e, s_r[src], np.float32(0.0))
            got[offs[j]:offs[j + 1]] = e
        results.append((out, got))
    return results


def run_generation(buckets: list, job_seed: int, generation: int, ht: bool,
                   masks: dict | None = None, r: int | None = None,
                   epp: int = MAX_PAYLOAD // ENTRY_BYTES, threads: int = 1,
                   return_wire: bool = False, bucket_id: int | None = None,
                   entry_masks: dict | None = None):
    """runner.py:211-276 hot-path composition with the channel replaced by
    ``masks``: ht -> RhtContext(derive_seed(seed, g%65536, g)) (:217-222),
    encode every node and cast float32 (:223-225), TAR (:230-246), decode
    per node with DropMask(received) and cast float32, EmptyReception ->
    zeros (:248-258).  rotation r = generation % n unless given (:274-275).

    ``threads`` > 1 runs the per-node encode/decode in a thread pool (numpy
    releases the GIL).  ``bucket_id`` replaces the runner's ``g % 65536`` in
    the seed derivation (a DDP hook keys the codec by its bucket index).
    """
    n = len(buckets)
    length = len(buckets[0])
    if r is None:
        r = generation % n
    pool = ThreadPoolExecutor(threads) if threads > 1 else None
    pmap = pool.map if pool else map
    try:
        if ht:
            dim = next_pow2(length)
            bid = generation % 65536 if bucket_id is None else bucket_id
            signs = rht_signs(dim, derive_seed(job_seed, bid, generation))
            wire = list(pmap(lambda b: rht_encode(b, dim, signs).astype(np.float32), buckets))
        else:
            dim = length
            wire = [np.asarray(b, dtype=np.float32) for b in buckets]
        if masks is None:
            masks = full_masks(dim, n, r, epp)
        tar = tar_masked(wire, r, masks, epp, entry_masks)
        if ht:
            def dec(res):
                entries, got = res
                try:
                    return rht_decode(entries, got, length, signs).astype(np.float32)
                except EmptyReception:
                    return np.zeros(length, dtype=np.float32)
            results = list(pmap(dec, tar))
        else:
            results = [e for e, _ in tar]
    finally:
        if pool:
            pool.shutdown()
    if return_wire:
        return results, wire, tar
    return results


# --------------------------------------------------------------------------
# workload  (harness.py)
# --------------------------------------------------------------------------


def bucket_rng(seed: int) -> np.random.Generator:
    """harness.py:67-71."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), 0x6275636B])))


def make_buckets(seed: int, n: int, length: int) -> list:
    """harness.py:117-120: n float32 standard-normal buckets, node order."""
    rng = bucket_rng(seed)
    return [rng.standard_normal(length).astype(np.float32) for _ in range(n)]


def oracle_allreduce(buckets: list) -> np.ndarray:
    """harness.py:30-38: exact float64 mean over node order."""
    acc = np.zeros(len(buckets[0]), dtype=np.float64)
    for b in buckets:
        acc += np.asarray(b, dtype=np.float64)
    return acc / len(buckets)
