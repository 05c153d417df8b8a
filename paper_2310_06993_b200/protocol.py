"""The reference's sans-IO collectives on device buffers.

``ubar.collectives`` (``/root/reference/pkg/src/ubar/collectives.py``)
expresses every AllReduce as a generator that yields channel commands
(``SendShard`` / ``OpenStage`` / ``AwaitStage`` / ``RoundEnd``) and receives
``StageResult``s back; a driver (in-memory, simulator or UDP) moves the data.
This module keeps that protocol -- same generator signatures, command types
and result types, so a reference caller's driver loop works unchanged -- with
the shards held as CUDA tensors and every arithmetic step in liboptr's
kernels:

* ``_mean_received`` (collectives.py:77-94) -> ``optr_mean_received`` (fp64,
  ascending node order, bit-identical);
* the ring's fp64 partial sums and masked all-gather (collectives.py:248-292)
  -> ``optr_ring_cast`` / ``optr_ring_step`` / ``optr_ring_finish``.

Drivers: ``run_lossless`` (collectives.py:321-401) and ``run_datagram``, the
UDP backend's drop model without sockets: every packet of ``max_payload``
bytes a sender transmits draws one coin from that sender's
``PCG64(SeedSequence([seed, rank]))`` stream in send order (datagram.py:
70-72,111-124), evaluated counter-indexed by liboptr, so any of the four
collectives reproduces the live backend's masks.  The batched fast paths
(``tar_allreduce_local``, ``TarCommunicator``) are what the gradient hot path
uses; this module is the reference-shaped entry point and the baselines
(Ring, PS, 2D TAR) for the MSE-ordering comparison.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, lib
from .schedule import PairSchedule, Topology, build_schedule, owned_shard
from .ubt import Completion, StageOutcome

ENTRY_BYTES = 4  # wire.py:23
MAX_PAYLOAD = 1400  # wire.py:22

__all__ = ["SendShard", "OpenStage", "AwaitStage", "RoundEnd", "StageResult", "AllReduceResult",
           "CollectiveDeadlock", "NodeStats", "tar_allreduce", "tar2d_allreduce", "ring_allreduce",
           "ps_allreduce", "run_lossless", "run_datagram", "shard_offsets", "shard_lengths"]


# ------------------------------------------------------------ commands
@dataclass
class SendShard:
    """collectives.py:25-34."""

    dst: int
    stage: str
    shard_index: int
    entry_offset: int
    data: object  # CUDA float32 tensor
    fan_in: int = 1


@dataclass
class OpenStage:
    """collectives.py:37-43: kind 1 = send/receive, 2 = broadcast/receive;
    expected: peer -> (shard_index, n_entries)."""

    key: str
    kind: int
    expected: dict


@dataclass
class AwaitStage:
    key: str


@dataclass
class RoundEnd:
    pass


@dataclass
class StageResult:
    """collectives.py:58-62: peer -> float32 data (zeros where missing),
    peer -> bool mask.  CUDA tensors."""

    outcome: StageOutcome
    data: dict
    mask: dict


@dataclass
class AllReduceResult:
    """collectives.py:65-74."""

    entries: object
    received: object


class CollectiveDeadlock(RuntimeError):
    pass


# ------------------------------------------------------------ helpers
def shard_lengths(length: int, n: int) -> list:
    """wire.py:121-126."""
    base, extra = divmod(int(length), n)
    return [base + 1 if j < extra else base for j in range(n)]


def shard_offsets(length: int, n: int) -> list:
    """wire.py:129-133."""
    offs = [0]
    for ln in shard_lengths(length, n):
        offs.append(offs[-1] + ln)
    return offs


def _torch():
    import torch

    return torch


class _Vec:
    """A node's entries on the device; remembers whether the caller gave numpy
    (results go back as numpy, like the reference's)."""

    def __init__(self, entries):
        torch = _torch()
        if isinstance(entries, torch.Tensor):
            if not entries.is_cuda:
                raise ValueError("torch tensors must live on a CUDA device")
            self.t = entries.detach().to(torch.float32).contiguous()
            self.numpy = False
        else:
            arr = np.ascontiguousarray(np.asarray(entries, dtype=np.float32))
            self.t = torch.from_numpy(arr).cuda()
            self.numpy = True

    def out(self, t):
        return t.cpu().numpy() if self.numpy else t


def _stream(t):
    return _torch().cuda.current_stream(t.device).cuda_stream


def _mean_received(rank: int, own, result: StageResult, n: int):
    """collectives.py:77-94 on the GPU (optr_mean_received): fp64 sum in
    ascending node order of own + each peer's zero-filled data, divided by
    1 + the peers' received flags; float32 result."""
    torch = _torch()
    own = own.to(torch.float32).contiguous()
    out = torch.empty_like(own)
    peers = (ctypes.c_void_p * n)()
    masks = (ctypes.c_void_p * n)()
    keep = []
    for i in range(n):
        if i != rank and i in result.data:
            d = result.data[i].contiguous()
            m = result.mask[i].to(torch.bool).contiguous()
            keep += [d, m]
            peers[i] = d.data_ptr() if d.numel() else None
            masks[i] = m.data_ptr() if m.numel() else None
    if own.numel():
        check(lib().optr_mean_received(own.data_ptr(), peers, masks, n, rank, own.numel(), out.data_ptr(),
                                       _stream(own)), "mean_received")
    return out


# ------------------------------------------------------------ collectives
def tar_allreduce(rank: int, entries, topo: Topology, r: int, schedule: PairSchedule):
    """Transpose AllReduce (collectives.py:97-150): stage 1 scatters shard
    owned_shard(dst) to every dst in schedule order and averages the own
    shard over what arrived; stage 2 broadcasts it; the result assembles
    every owner's shard, zero-filled where missing."""
    torch = _torch()
    n = topo.n
    v = _Vec(entries)
    x = v.t
    offs = shard_offsets(len(x), n)
    my_j = owned_shard(rank, r, n)

    def shard_of(j):
        return x[offs[j]:offs[j + 1]]

    yield OpenStage("s1", 1, {p: (my_j, offs[my_j + 1] - offs[my_j]) for p in range(n) if p != rank})
    for rnd in schedule.rounds:
        dsts = rnd[rank]
        for dst in dsts:
            j = owned_shard(dst, r, n)
            yield SendShard(dst, "s1", j, offs[j], shard_of(j), fan_in=len(dsts))
        yield RoundEnd()
    res1 = yield AwaitStage("s1")
    s_r = _mean_received(rank, shard_of(my_j), res1, n)

    expected2 = {}
    for p in range(n):
        if p != rank:
            j = owned_shard(p, r, n)
            expected2[p] = (j, offs[j + 1] - offs[j])
    yield OpenStage("s2", 2, expected2)
    for rnd in schedule.rounds:
        dsts = rnd[rank]
        for dst in dsts:
            yield SendShard(dst, "s2", my_j, offs[my_j], s_r, fan_in=len(dsts))
        yield RoundEnd()
    res2 = yield AwaitStage("s2")

    out = torch.zeros_like(x)
    got = torch.zeros(len(x), dtype=torch.bool, device=x.device)
    out[offs[my_j]:offs[my_j + 1]] = s_r
    got[offs[my_j]:offs[my_j + 1]] = True
    for p in range(n):
        if p != rank:
            j = owned_shard(p, r, n)
            out[offs[j]:offs[j + 1]] = res2.data[p]
            got[offs[j]:offs[j + 1]] = res2.mask[p]
    return AllReduceResult(v.out(out), v.out(got))


def _relabel(res: StageResult, order: list) -> StageResult:
    return StageResult(res.outcome, {order.index(p): d for p, d in res.data.items()},
                       {order.index(p): m for p, m in res.mask.items()})


def tar2d_allreduce(rank: int, entries, topo: Topology, r: int):
    """Hierarchical TAR (collectives.py:153-245): intra-group stage 1,
    inter-group mean of each shard among the ranks holding it, intra-group
    broadcast."""
    torch = _torch()
    n = topo.n
    g = topo.group_size or n
    groups = n // g
    gid, lid = divmod(rank, g)
    members = [gid * g + m for m in range(g)]
    rank_peers = [q * g + lid for q in range(groups)]
    v = _Vec(entries)
    x = v.t
    offs = shard_offsets(len(x), g)
    my_j = owned_shard(lid, r, g)

    def shard_of(j):
        return x[offs[j]:offs[j + 1]]

    if g > 1:  # phase 1: intra-group send/receive + mean
        sched = build_schedule(g, 1)
        yield OpenStage("p1", 1, {members[p]: (my_j, offs[my_j + 1] - offs[my_j]) for p in range(g) if p != lid})
        for rnd in sched.rounds:
            for ldst in rnd[lid]:
                j = owned_shard(ldst, r, g)
                yield SendShard(members[ldst], "p1", j, offs[j], shard_of(j), fan_in=1)
            yield RoundEnd()
        res = yield AwaitStage("p1")
        local = _mean_received(lid, shard_of(my_j), _relabel(res, members), g)
    else:
        local = shard_of(my_j).clone()

    if groups > 1:  # phase 2: inter-group, rank-wise
        sched = build_schedule(groups, 1)
        ln = offs[my_j + 1] - offs[my_j]
        yield OpenStage("p2", 1, {rank_peers[q]: (my_j, ln) for q in range(groups) if q != gid})
        for rnd in sched.rounds:
            for qdst in rnd[gid]:
                yield SendShard(rank_peers[qdst], "p2", my_j, offs[my_j], local, fan_in=1)
            yield RoundEnd()
        res = yield AwaitStage("p2")
        global_shard = _mean_received(gid, local, _relabel(res, rank_peers), groups)
    else:
        global_shard = local

    out = torch.zeros_like(x)
    got = torch.zeros(len(x), dtype=torch.bool, device=x.device)
    out[offs[my_j]:offs[my_j + 1]] = global_shard
    got[offs[my_j]:offs[my_j + 1]] = True
    if g > 1:  # phase 3: intra-group broadcast
        sched = build_schedule(g, 1)
        expected = {}
        for m in range(g):
            if m != lid:
                j = owned_shard(m, r, g)
                expected[members[m]] = (j, offs[j + 1] - offs[j])
        yield OpenStage("p3", 2, expected)
        for rnd in sched.rounds:
            for ldst in rnd[lid]:
                yield SendShard(members[ldst], "p3", my_j, offs[my_j], global_shard, fan_in=1)
            yield RoundEnd()
        res = yield AwaitStage("p3")
        for m in range(g):
            if m != lid:
                j = owned_shard(m, r, g)
                out[offs[j]:offs[j + 1]] = res.data[members[m]]
                got[offs[j]:offs[j + 1]] = res.mask[members[m]]
    return AllReduceResult(v.out(out), v.out(got))


def ring_allreduce(rank: int, entries, topo: Topology):
    """Ring reduce-scatter + all-gather (collectives.py:248-292): fp64 partial
    sums travel hop by hop (a dropped chunk is missing downstream, by
    design); the all-gather keeps the partial value where a chunk dropped."""
    torch = _torch()
    n = topo.n
    v = _Vec(entries)
    x = v.t
    offs = shard_offsets(len(x), n)
    buf = x.double()
    prev, nxt = (rank - 1) % n, (rank + 1) % n

    def chunk(j):
        return buf[offs[j]:offs[j + 1]]

    def as_f32(j):
        c = chunk(j)
        f = torch.empty(c.numel(), dtype=torch.float32, device=c.device)
        if c.numel():
            check(lib().optr_ring_cast(c.data_ptr(), c.numel(), f.data_ptr(), _stream(c)), "ring_cast")
        return f

    for k in range(n - 1):
        send_j, recv_j = (rank - k) % n, (rank - k - 1) % n
        key = f"rs{k}"
        yield OpenStage(key, 1, {prev: (recv_j, offs[recv_j + 1] - offs[recv_j])})
        yield SendShard(nxt, key, send_j, offs[send_j], as_f32(send_j), fan_in=1)
        res = yield AwaitStage(key)
        c = chunk(recv_j)
        if c.numel():  # missing entries add zero
            d = res.data[prev].contiguous()
            check(lib().optr_ring_step(c.data_ptr(), d.data_ptr(), None, c.numel(), 0, _stream(c)), "ring_step")
        yield RoundEnd()
    for k in range(n - 1):
        send_j, recv_j = (rank + 1 - k) % n, (rank - k) % n
        key = f"ag{k}"
        yield OpenStage(key, 2, {prev: (recv_j, offs[recv_j + 1] - offs[recv_j])})
        yield SendShard(nxt, key, send_j, offs[send_j], as_f32(send_j), fan_in=1)
        res = yield AwaitStage(key)
        c = chunk(recv_j)
        if c.numel():  # keep the partial value where dropped
            d = res.data[prev].contiguous()
            m = res.mask[prev].to(torch.bool).contiguous()
            check(lib().optr_ring_step(c.data_ptr(), d.data_ptr(), m.data_ptr(), c.numel(), 1, _stream(c)),
                  "ring_step")
        yield RoundEnd()
    out = torch.empty(len(x), dtype=torch.float32, device=x.device)
    if len(x):
        check(lib().optr_ring_finish(buf.data_ptr(), n, len(x), out.data_ptr(), _stream(buf)), "ring_finish")
    return AllReduceResult(v.out(out), v.out(torch.ones(len(x), dtype=torch.bool, device=x.device)))


def ps_allreduce(rank: int, entries, topo: Topology, server: int):
    """Parameter server (collectives.py:295-314): full-incast gather and
    mean at `server`, broadcast back."""
    torch = _torch()
    n = topo.n
    v = _Vec(entries)
    x = v.t
    ln = len(x)
    if rank == server:
        yield OpenStage("gather", 1, {p: (0, ln) for p in range(n) if p != server})
        res = yield AwaitStage("gather")
        mean = _mean_received(rank, x, res, n)
        for dst in range(n):
            if dst != server:
                yield SendShard(dst, "bcast", 0, 0, mean, fan_in=1)
        yield RoundEnd()
        return AllReduceResult(v.out(mean), v.out(torch.ones(ln, dtype=torch.bool, device=x.device)))
    yield OpenStage("bcast", 2, {server: (0, ln)})
    yield SendShard(server, "gather", 0, 0, x, fan_in=n - 1)
    yield RoundEnd()
    res = yield AwaitStage("bcast")
    return AllReduceResult(v.out(res.data[server].clone()), v.out(res.mask[server].clone()))


# ------------------------------------------------------------ drivers
@dataclass
class NodeStats:
    """Per-node channel accounting (simdriver.py:26-45)."""

    bytes_sent: int = 0
    bytes_received: int = 0
    bytes_expected: int = 0
    outcomes: list = field(default_factory=list)  # (key, kind, StageOutcome)
    result: object = None

    @property
    def loss_rate(self) -> float:
        return 0.0 if self.bytes_expected == 0 else 1.0 - self.bytes_received / self.bytes_expected

    @property
    def timeout_occurred(self) -> bool:
        return any(o.completion is not Completion.ON_TIME for _, _, o in self.outcomes)


def _drive(generators: list, deliver):
    """The reference driver loop (collectives.py:321-401): each send lands in
    the destination's stage immediately (through ``deliver``), a stage
    completes once every expected peer has sent.  Returns (results, stats)."""
    torch = _torch()
    n = len(generators)
    results: list = [None] * n
    stats = [NodeStats() for _ in range(n)]
    done = [False] * n
    stages: dict = {}
    waiting: dict = {}
    pending: dict = {i: None for i in range(n)}

    def stage(dst, key):
        return stages.setdefault((dst, key), {"expected": None, "kind": 1, "data": {}, "mask": {}})

    def complete(dst, key):
        st = stage(dst, key)
        return st["expected"] is not None and all(p in st["data"] for p in st["expected"])

    def result_for(dst, key):
        st = stages[(dst, key)]
        data, mask, exp_b, got_b = {}, {}, 0, 0
        for p, (_j, cnt) in st["expected"].items():
            data[p] = st["data"][p]
            mask[p] = st["mask"][p]
            exp_b += cnt * ENTRY_BYTES
            got_b += int(mask[p].sum().item()) * ENTRY_BYTES
        out = StageOutcome(completion=Completion.ON_TIME, elapsed=0.0,
                           loss_rate=(1.0 - got_b / exp_b) if exp_b else 0.0,
                           expected_bytes=exp_b, received_bytes=got_b, last_pct_from_all=True)
        stats[dst].bytes_expected += exp_b
        stats[dst].bytes_received += got_b
        stats[dst].outcomes.append((key, st["kind"], out))
        return StageResult(out, data, mask)

    while not all(done):
        progress = False
        for i, gen in enumerate(generators):
            if done[i]:
                continue
            if i in waiting:
                if not complete(i, waiting[i]):
                    continue
                pending[i] = result_for(i, waiting.pop(i))
            while True:
                try:
                    cmd = gen.send(pending[i])
                except StopIteration as stop:
                    results[i] = stop.value
                    stats[i].result = stop.value
                    done[i] = True
                    progress = True
                    break
                pending[i] = None
                if isinstance(cmd, SendShard):
                    data = cmd.data.to(torch.float32).contiguous()
                    d, m = deliver(i, cmd.dst, data)
                    stats[i].bytes_sent += data.numel() * ENTRY_BYTES
                    st = stage(cmd.dst, cmd.stage)
                    st["data"][i], st["mask"][i] = d, m
                elif isinstance(cmd, OpenStage):
                    st = stage(i, cmd.key)
                    st["expected"], st["kind"] = cmd.expected, cmd.kind
                elif isinstance(cmd, RoundEnd):
                    pass
                elif isinstance(cmd, AwaitStage):
                    if complete(i, cmd.key):
                        pending[i] = result_for(i, cmd.key)
                        continue
                    waiting[i] = cmd.key
                    progress = True
                    break
                else:
                    raise TypeError(f"unknown channel command {cmd!r}")
        if not progress:
            stuck = {i: waiting.get(i) for i in range(n) if not done[i]}
            raise CollectiveDeadlock(f"no progress; nodes blocked on {stuck}")
    return results, stats


def run_lossless(generators: list) -> list:
    """collectives.py:321-401: a perfect channel; every send delivered whole
    (a device copy)."""
    torch = _torch()

    def deliver(_src, _dst, data):
        return data.clone(), torch.ones(data.numel(), dtype=torch.bool, device=data.device)

    return _drive(generators, deliver)[0]


def run_datagram(generators: list, seed: int, drop_prob: float, max_payload: int = MAX_PAYLOAD,
                 stream_offsets=None, return_stats: bool = False):
    """The UDP backend's seeded send-side drop model (datagram.py:70-72,
    111-124) without sockets or timeouts: sender ``src`` cuts each send into
    packets of ``max_payload // 4`` entries and draws one coin per packet, in
    send order, from ``PCG64(SeedSequence([seed, src]))`` (only when
    ``drop_prob > 0``, datagram.py:122); a dropped packet's entries arrive as
    zeros with their flags cleared.  ``stream_offsets``: draws each sender's
    stream made before (a reused endpoint).  Returns the results (and the
    per-node ``NodeStats`` with ``return_stats``)."""
    from .collectives import coin_packets

    torch = _torch()
    epp = max_payload // ENTRY_BYTES
    if epp <= 0:
        raise ValueError("max_payload must hold at least one entry")
    ctr = [int(v) for v in stream_offsets] if stream_offsets is not None else [0] * len(generators)

    def deliver(src, _dst, data):
        ne = data.numel()
        npk = -(-ne // epp) if ne else 0
        if drop_prob <= 0 or npk == 0:
            return data.clone(), torch.ones(ne, dtype=torch.bool, device=data.device)
        keep = coin_packets(seed, src, ctr[src], npk, drop_prob)
        ctr[src] += npk
        m = torch.from_numpy(np.repeat(keep, epp)[:ne]).to(data.device)
        return torch.where(m, data, torch.zeros((), device=data.device)), m

    results, stats = _drive(generators, deliver)
    return (results, stats) if return_stats else results
