"""One TAR worker per GPU (NVLink peer pulls) against the oracle.

Spawns one process per GPU (NCCL for the plumbing, like torchrun) and
compares every rank's result with the oracle's n-worker generation under
the same coin masks.  The CPU-only test exercises the host-side handle
exchange over gloo with world_size 2.
"""

import os
import socket
import tempfile

import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")


def _world():
    """Ranks for the multi-GPU tests: one per GPU (<= 8), or OPTR_TEST_WORLD
    ranks round-robin over the GPUs (e.g. 8 ranks on 4 GPUs, with
    OPTR_FUSED_GRID capping each persistent grid so two fit on a GPU)."""
    env = os.environ.get("OPTR_TEST_WORLD")
    return int(env) if env else min(torch.cuda.device_count(), 8)


def _dev(rank):
    return rank % torch.cuda.device_count()


def _init(rank, world, dev):
    """NCCL with one rank per GPU; gloo (host-side handle exchange only) when
    ranks share GPUs, which NCCL refuses.  A protocol deadlock in the fused
    kernel should fail the test in seconds, not hang it (watchdog)."""
    import torch.distributed as dist

    os.environ.setdefault("OPTR_WATCHDOG_S", "30")
    if world > torch.cuda.device_count():
        dist.init_process_group("gloo", rank=rank, world_size=world)
    else:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)


def _free_port():
    """A bindable port outside the ephemeral range (bind-to-0 ports can be
    taken again by the previous spawn's lingering NCCL / gloo sockets)."""
    import random

    for _ in range(200):
        p = random.randint(20000, 29999)
        s = socket.socket()
        try:
            s.bind(("127.0.0.1", p))
            return p
        except OSError:
            continue
        finally:
            s.close()
    raise RuntimeError("no free port")


# ------------------------------------------------------------ CPU / gloo
def _gloo_worker(rank, world, port, outdir):
    import torch.distributed as dist

    from paper_2310_06993_b200.dist import all_gather_bytes

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank] * 7 + [255 - rank])
    got = all_gather_bytes(blob)
    np.save(os.path.join(outdir, f"r{rank}.npy"), np.frombuffer(b"".join(got), dtype=np.uint8))
    dist.destroy_process_group()


def test_handle_exchange_gloo_world2():
    import torch.multiprocessing as mp

    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        want = b"".join(bytes([r] * 7 + [255 - r]) for r in range(world))
        for r in range(world):
            assert np.load(os.path.join(d, f"r{r}.npy")).tobytes() == want


# ------------------------------------------------------------ multi-GPU
CASES = [
    # L, p, gen, ht, dtype
    (1 << 16, 0.05, 3, True, "f32"),
    (100_000, 0.01, 5, True, "f32"),
    (25_000_000, 0.01, 1, True, "f32"),
    (12_345, 0.05, 2, False, "f32"),
    (1 << 20, 0.02, 4, True, "bf16"),
    # fused multi-GPU kernel (D = 2^23, 2^25): against the oracle / exact mean
    (5_000_000, 0.02, 6, True, "f32"),
    (4_200_000, 0.01, 7, True, "bf16"),
    (25_000_000, 0.0, 2, True, "f32"),
]


def _gpu_worker(rank, world, port, outdir):
    import torch.distributed as dist

    from paper_2310_06993_b200.collectives import MaskSpec
    from paper_2310_06993_b200.dist import TarCommunicator

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(_dev(rank))
    dev = torch.device("cuda", _dev(rank))
    _init(rank, world, dev)
    comm = TarCommunicator(max_len=max(c[0] for c in CASES))
    for ci, (L, p, gen, ht, dt) in enumerate(CASES):
        buckets = O.make_buckets(100 + ci, world, L)
        x = torch.from_numpy(buckets[rank]).to(dev)
        if dt == "bf16":
            x = x.to(torch.bfloat16)
        out = torch.empty(L, dtype=torch.float32, device=dev)
        rec = torch.zeros(2, dtype=torch.int64, device=dev)
        comm.allreduce(x, out, rotation=gen % world, ht=ht, job_seed=9, generation=gen,
                       masks=MaskSpec.coin(700 + ci, p), received=rec)
        torch.cuda.synchronize()
        np.save(os.path.join(outdir, f"c{ci}_r{rank}.npy"), out.cpu().numpy())
        np.save(os.path.join(outdir, f"c{ci}_r{rank}_rec.npy"), rec.cpu().numpy())
        if dt == "bf16":  # bf16 out as well (DDP's bf16 buckets): the decode's bf16 TMA store
            out16 = torch.empty(L, dtype=torch.bfloat16, device=dev)
            comm.allreduce(x, out16, rotation=gen % world, ht=ht, job_seed=9, generation=gen,
                           masks=MaskSpec.coin(700 + ci, p))
            torch.cuda.synchronize()
            np.save(os.path.join(outdir, f"c{ci}_r{rank}_bf16.npy"), out16.float().cpu().numpy())
    comm.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.multigpu
def test_tar_rht_multi_gpu_vs_oracle():
    import torch.multiprocessing as mp

    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = _world()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gpu_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for ci, (L, p, gen, ht, dt) in enumerate(CASES):
            buckets = O.make_buckets(100 + ci, world, L)
            if dt == "bf16":
                buckets = [torch.from_numpy(b).to(torch.bfloat16).float().numpy() for b in buckets]
            r = gen % world
            dim = O.next_pow2(L) if ht else L
            masks = O.datagram_masks(700 + ci, dim, world, r, p)
            if L > 5_000_000:
                # size-independent checks at the headline size: counts bit-exact,
                # lossless-ish agreement with the exact mean bounded by the loss
                mean = O.oracle_allreduce(buckets)
                sc = O.stage_counts(masks, dim, world, r, 350)
                for rank in range(world):
                    out = np.load(os.path.join(d, f"c{ci}_r{rank}.npy")).astype(np.float64)
                    rec = np.load(os.path.join(d, f"c{ci}_r{rank}_rec.npy"))
                    assert rec[0] == sc[(1, rank)][0] and rec[1] == sc[(2, rank)][0]
                    rel = np.linalg.norm(out - mean) / np.linalg.norm(mean)
                    assert rel < (1e-5 if p == 0 else 0.3), (ci, rank, rel)
                continue
            want = O.run_generation(buckets, 9, gen, ht, masks=masks, r=r)
            for rank in range(world):
                if dt == "bf16":
                    o16 = np.load(os.path.join(d, f"c{ci}_r{rank}_bf16.npy")).astype(np.float64)
                    assert np.linalg.norm(o16 - want[rank]) / np.linalg.norm(want[rank]) < 1e-2, (ci, rank)
                out = np.load(os.path.join(d, f"c{ci}_r{rank}.npy"))
                if ht:
                    rel = np.linalg.norm(out.astype(np.float64) - want[rank]) / np.linalg.norm(want[rank])
                    assert rel < 1e-5, (ci, rank, rel)
                else:
                    np.testing.assert_array_equal(out, want[rank])


# ------------------------------------------------------------ DDP hook
def _ddp_worker(rank, world, port, outdir):
    import torch.distributed as dist
    import torch.nn as nn
    from torch.nn.parallel import DistributedDataParallel as DDP

    from paper_2310_06993_b200.ddp_hook import OptiReduceState, max_bucket_len_for, optireduce_hook

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(_dev(rank))
    dev = torch.device("cuda", _dev(rank))
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    grads = {}
    big = os.environ.get("OPTR_TEST_DDP_BIG") == "1"
    for mode in ("nccl", "overlap", "ordered"):
        torch.manual_seed(0)
        if big:  # one 6.55M-entry bucket (D = 2^23): the fused multi-GPU kernel
            model = nn.Sequential(nn.Linear(512, 2560, bias=False), nn.ReLU(), nn.Linear(2560, 2560),
                                  nn.ReLU(), nn.Linear(2560, 10)).to(dev)
        else:
            model = nn.Sequential(nn.Linear(512, 1024), nn.ReLU(), nn.Linear(1024, 700), nn.ReLU(),
                                  nn.Linear(700, 10)).to(dev)
        ddp = DDP(model, device_ids=[rank], bucket_cap_mb=25 if big else 1)
        if mode != "nccl":
            state = OptiReduceState(max_bucket_len=max_bucket_len_for(model, 1), ht=True, seed=3,
                                    overlap=(mode == "overlap"))
            ddp.register_comm_hook(state, optireduce_hook)
        g = torch.Generator(device=dev).manual_seed(100 + rank)
        for _step in range(2):  # second pass reuses the buffers at the next generation
            model.zero_grad(set_to_none=True)
            x = torch.randn(64, 512, device=dev, generator=g)
            loss = ddp(x).square().mean()
            loss.backward()
        torch.cuda.synchronize()
        grads[mode] = torch.cat([p.grad.flatten() for p in model.parameters()]).cpu().numpy()
        if mode != "nccl":
            assert state.generation == 2
            assert len(state.received) >= 2 and not state._pending
            state.comm.close()
    np.save(os.path.join(outdir, f"ddp_r{rank}.npy"), np.stack([grads["nccl"], grads["overlap"], grads["ordered"]]))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("big", [False, True])
def test_ddp_comm_hook_lossless_matches_mean(big, monkeypatch):
    """Lossless TAR+RHT through the DDP hook == DDP's own mean all-reduce
    within the float32 codec error (small buckets: the barrier path; one
    25 MB-class bucket: the fused kernel)."""
    import torch.multiprocessing as mp

    monkeypatch.setenv("OPTR_TEST_DDP_BIG", "1" if big else "0")

    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = _world()
    if world > torch.cuda.device_count():
        pytest.skip("DDP over NCCL needs one rank per GPU")
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_ddp_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        for r in range(world):
            ref, ovl, ordered = np.load(os.path.join(d, f"ddp_r{r}.npy"))
            for got in (ovl, ordered):
                rel = np.linalg.norm(got.astype(np.float64) - ref) / np.linalg.norm(ref)
                assert rel < 1e-5, rel
            np.testing.assert_array_equal(ovl, ordered)  # same kernels, same order of arithmetic


# ------------------------------------------- fused kernel vs barrier path
def _seq_worker(rank, world, port, outdir, fused):
    os.environ["OPTR_FUSED"] = "1" if fused else "0"
    import torch.distributed as dist

    from paper_2310_06993_b200.collectives import MaskSpec
    from paper_2310_06993_b200.dist import TarCommunicator

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(_dev(rank))
    dev = torch.device("cuda", _dev(rank))
    _init(rank, world, dev)
    lens = [5_000_000, 8_388_608, 3_000_000, 16_000_000, 5_000_000]
    comm = TarCommunicator(max_len=max(lens))
    g = torch.Generator(device=dev).manual_seed(50 + rank)
    xs = [torch.randn(L, device=dev, generator=g) for L in lens]
    outs = [torch.empty_like(x) for x in xs]
    recs = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in lens]
    for rep in range(2):  # second pass: both parities reused at the next epochs
        for b, L in enumerate(lens):
            gen = rep * len(lens) + b
            comm.allreduce(xs[b], outs[b], rotation=gen % world, ht=True, job_seed=4, generation=gen,
                           masks=MaskSpec.coin(300 + gen, 0.02), received=recs[b], async_op=True)
        comm.join()
    torch.cuda.synchronize()
    for b in range(len(lens)):
        np.save(os.path.join(outdir, f"f{int(fused)}_b{b}_r{rank}.npy"), outs[b].cpu().numpy())
        np.save(os.path.join(outdir, f"f{int(fused)}_b{b}_r{rank}_rec.npy"), recs[b].cpu().numpy())
    comm.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.multigpu
def test_fused_kernel_matches_barrier_path_async():
    """Async back-to-back buckets through the fused per-tile-flag kernel give
    the barrier-separated path's results (float32 codec tolerance; the pass
    order differs) and identical received counts."""
    import torch.multiprocessing as mp

    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = _world()
    with tempfile.TemporaryDirectory() as d:
        for fused in (True, False):
            mp.spawn(_seq_worker, args=(world, _free_port(), d, fused), nprocs=world, join=True)
        for b in range(5):
            for r in range(world):
                a = np.load(os.path.join(d, f"f1_b{b}_r{r}.npy")).astype(np.float64)
                c = np.load(os.path.join(d, f"f0_b{b}_r{r}.npy")).astype(np.float64)
                assert np.linalg.norm(a - c) / np.linalg.norm(c) < 1e-5, (b, r)
                np.testing.assert_array_equal(np.load(os.path.join(d, f"f1_b{b}_r{r}_rec.npy")),
                                              np.load(os.path.join(d, f"f0_b{b}_r{r}_rec.npy")))
