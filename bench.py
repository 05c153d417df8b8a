"""Benchmark of the TAR+RHT gradient-aggregation hot path (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload resnet50|headline|bert|gpt2xl|cfg1] [--workers n]

A *step* is one Transpose-AllReduce generation over every bucket of the
workload's gradient (RHT encode -> stage-1 masked mean -> stage-2 gather ->
masked RHT decode), 1% seeded datagram-coin drops unless ``--drop`` says
otherwise.  At ``--gpus 1`` the ``--workers`` (default 4, the reference's
``SimSession`` shape, BASELINE configs[0]) workers are co-resident on one GPU;
at ``--gpus N>1`` there is one worker per GPU (torchrun, NVLink peer pulls).

``value``: whole-job gradient GB/s reduced = workers * bytes(gradient) / step
time (device time, CUDA events, max over ranks).  ``e2e``: the same through
the public API with pinned host buffers copied in and results copied out
inside the timed region, pipelined per bucket (bucket b's D2H overlaps bucket
b+1's H2D).  ``roofline``: the dominant kernel's algorithmic
bytes / its live CUDA-event duration against MEASURED_PEAKS.json.
``cpu_baseline``: the reference algorithm (oracle port of ubar, numpy, the
same masks) timed on this host on one bucket.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MB25 = 25 * 1024 * 1024 // 4  # 25 MB fp32 bucket = 6,553,600 entries
WORKLOADS = {
    # name: (total entries, bucket entries, input dtype, description)
    "resnet50": (25_557_032, MB25, "f32", "ResNet-50 gradient (25.6M fp32) in 25 MB buckets"),
    "headline": (25_000_000, 25_000_000, "f32", "one 25M-entry fp32 bucket (north-star headline)"),
    "bert": (340_000_000, MB25, "f32", "BERT-large gradient (340M fp32) in 25 MB buckets"),
    "gpt2xl": (1_557_611_200, 25 * 1024 * 1024 // 2, "bf16",
               "GPT-2 XL gradient (1.56B bf16 in / fp32 aggregate) in 25 MB bf16 buckets"),
    "cfg1": (1_048_576, 1_048_576, "f32", "one 1M-entry fp32 bucket (BASELINE configs[0])"),
}


def bucket_sizes(total: int, per: int) -> list:
    out = [per] * (total // per)
    if total % per:
        out.append(total % per)
    return out


def next_pow2(n: int) -> int:
    return 1 if n <= 1 else 1 << (n - 1).bit_length()


def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "src": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "src": "fallback"}


NVLINK_GBS = 770.0  # measured single-peer SM pull, GB/s per direction (profiles/r02_nvlink_probe_2gpu.jsonl)
# every GPU pulling from every peer at once (the TAR exchange pattern), GB/s in
# per GPU, wall clock (profiles/r02_nvlink_probe_{2,4}gpu.jsonl); the roofline's
# NVLink denominator where measured, else the single-peer figure
NVLINK_ALLPEER_GBS = {2: 646.1, 4: 606.4}


def nvlink_peak(n: int) -> float:
    return NVLINK_ALLPEER_GBS.get(n, NVLINK_GBS)


# ------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ roofline
def kernel_bytes(cls: str, dim: int, L: int, n: int, s_in: int, s_out: int) -> int:
    """Algorithmic HBM bytes of one launch of a kernel class for ONE worker
    (DESIGN.md "Kernels"): reads + writes each counted once."""
    Y = 4 * dim
    S = Y // n
    return {
        "enc_first": s_in * L + Y,     # read x, write the first-pass wire
        "enc_mid": 2 * Y,
        "enc_last": 2 * Y,             # read + write the wire in place
        "aggregate": n * S + S,        # n shard copies in, one mean out
        "dec_first": Y + Y,            # gather n aggregates, write scratch
        "dec_mid": 2 * Y,
        "dec_last": Y + s_out * L,     # read scratch, write output
        "assemble": Y + s_out * L,
        "prep": dim // 8,
        # one GPU: last encode pass of every worker + stage-1 mean, per
        # worker: read its first-pass vector, write 1/n of the aggregate
        "enc_mean": Y + S,
        # multi-GPU fused kernel: contiguous encode pass in place (2Y), owner
        # shard in from n wire vectors + mean out to n receive vectors (local
        # side only: S in, S out), contiguous decode pass in place (2Y)
        "fused": 4 * Y + 2 * S,
        # multi-GPU small-bucket kernel (the whole call in one launch): x in,
        # four in-place passes over the wire vector, owner shard in + mean
        # out, stage-2 receive written to the wire vector, out
        "small": s_in * L + 8 * Y + 2 * S + Y + s_out * L,
    }.get(cls, 0)


def step_alg_bytes(buckets, n_workers, s_in, s_out, ht):
    """HBM_alg per worker per step, and NVLink bytes."""
    hbm = 0
    nvl = 0
    for L in buckets:
        if ht:
            Y = 4 * next_pow2(L)
            hbm += (s_in + s_out) * L + 3 * Y + Y // n_workers
            nvl += 2 * Y * (n_workers - 1) // n_workers
        else:
            hbm += s_in * L + 4 * L // n_workers + 4 * L + s_out * L
            nvl += 2 * 4 * L * (n_workers - 1) // n_workers
    return hbm, nvl


# kernel classes -> kernel names in the one-GPU ncu capture (decode order there:
# strided gather first, contiguous last)
NCU_NAMES = {  # regexes for the one-GPU fast plan (stage count free: it depends on the tile shape)
    "enc_first": r"tma_pass_kernel<\d+, \d, 1, 1,",
    "enc_mean": r"tma_mean_kernel",
    "dec_first": r"tma_gather_shared_kernel|tma_pass_kernel<\d+, \d, 0, 2,",
    "dec_last": r"tma_pass_kernel<\d+, \d, 1, 0, SnkDecode",
    "aggregate": r"tma_agg_kernel",
    "prep": r"prep_kernel",
}


def ncu_traffic(cls: str, multi: bool):
    """(dram read+write bytes per launch of `cls`, source file) from profiles/, or None."""
    if multi:
        return None
    import glob

    # the newest capture of the current kernels
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_1gpu_fastplan.json")))
    if not files or cls not in NCU_NAMES:
        return None
    try:
        with open(files[-1]) as fh:
            entries = json.load(fh)
        for e in entries:
            if re.search(NCU_NAMES[cls], e["kernel"]):
                rd, wr = float(e["dram__bytes_read.sum"]), float(e["dram__bytes_write.sum"])
                scale = 1e6 if rd + wr < 1e5 else 1.0  # the raw page reports MB
                return int((rd + wr) * scale), os.path.basename(files[-1])
    except Exception:
        return None
    return None


# ------------------------------------------------------------ CPU baseline
def cpu_baseline(bucket_len: int, n_workers: int, drop: float, ht: bool, threads: int):
    """The reference algorithm (oracle = numpy restatement of ubar's
    rht_encode / _mean_received / assembly / rht_decode) on one bucket with
    the same coin masks.  Returns (GB/s of gradient reduced, seconds)."""
    import numpy as np

    import oracle as O

    buckets = O.make_buckets(0, n_workers, bucket_len)
    dim = next_pow2(bucket_len) if ht else bucket_len
    t0 = time.perf_counter()
    masks = O.datagram_masks(12345, dim, n_workers, 0, drop)
    O.run_generation(buckets, 0, 0, ht, masks=masks, r=0, threads=threads)
    dt = time.perf_counter() - t0
    return n_workers * 4 * bucket_len / dt / 1e9, dt


# ------------------------------------------------------------ our arm
def run_ours(args):
    import torch

    from paper_2310_06993_b200 import _lib
    from paper_2310_06993_b200.collectives import MaskSpec, local_join, tar_allreduce_local

    total, per, dt_name, desc = WORKLOADS[args.workload]
    dtype = torch.bfloat16 if dt_name == "bf16" else torch.float32
    s_in = 2 if dt_name == "bf16" else 4
    s_out = s_in
    buckets = bucket_sizes(total, per)
    ht = args.ht == "on"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    multi = world > 1
    n_workers = world if multi else args.workers

    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    if multi:
        import torch.distributed as dist

        from paper_2310_06993_b200.dist import TarCommunicator

        dist.init_process_group("nccl", device_id=dev)
        comm = TarCommunicator(max_len=max(buckets), epp=350)
        grads = [torch.randn(L, device=dev, generator=g).to(dtype) for L in buckets]
        outs = [torch.empty_like(x) for x in grads]
    else:
        grads = [[torch.randn(L, device=dev, generator=g).to(dtype) for _ in range(n_workers)]
                 for L in buckets]
        outs = [[torch.empty_like(x) for x in ws] for ws in grads]
    stream = torch.cuda.current_stream(dev)
    drop = args.drop
    state = {"gen": 0}
    overlap = True  # pass (A): buckets pipelined two in flight

    def call_bucket(b, gen, src, dst, async_op):
        masks = MaskSpec.coin(1000003 * gen + b, drop) if drop > 0 else MaskSpec.none()
        r = gen % n_workers
        if multi:
            comm.allreduce(src[b], dst[b], rotation=r, ht=ht, job_seed=7,
                           generation=gen, bucket_id=b, masks=masks, async_op=async_op)
        else:
            tar_allreduce_local(src[b], rotation=r, ht=ht, job_seed=7, generation=gen,
                                bucket_id=b, masks=masks, out=dst[b], async_op=async_op)

    def one_step(src=None, dst=None, overlap=True):
        gen = state["gen"]
        for b in range(len(buckets)):
            call_bucket(b, gen, src or grads, dst or outs, overlap)
        if multi:
            comm.join()
        else:
            local_join()
        state["gen"] += 1

    def barrier():
        if multi:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if not multi:
            return v
        import torch.distributed as dist

        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(overlap: bool, kernel_events: bool):
        """K steps between a barrier + synchronize on both sides, CUDA events
        on the calling stream; optionally every library launch bracketed by
        its own events (optr_timing_*).  Returns (ms per step over ranks,
        per-kernel {class: (ms, launches, worker-passes)}, launches)."""
        barrier()
        _lib.timing_collect()
        _lib.timing_enable(kernel_events)
        launches0 = _lib.launch_count()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            one_step(overlap=overlap)
        ev1.record(stream)
        torch.cuda.synchronize()
        launches = _lib.launch_count() - launches0
        _lib.timing_enable(False)
        per = _lib.timing_collect()
        return max_over_ranks(ev0.elapsed_time(ev1)) / args.steps, per, launches

    # ---- device-timed steps
    for _ in range(args.warmup):
        one_step(overlap=overlap)
    barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    # (A) the headline: buckets pipelined two in flight, as a DDP comm hook runs them
    ms_per_step, _unused, launches = timed(overlap, False)
    # (B) the same with every launch bracketed by CUDA events: per-kernel times
    #     under the two-bucket concurrency (contended: they overlap each other)
    ms_events, per_contended, _l = timed(overlap, True)
    # (C) buckets serialised, every launch bracketed: isolated per-kernel times,
    #     the roofline's denominators
    ms_serial, per_kernel, _l = timed(False, True)
    clk = clocks.stop()

    grad_bytes = s_in * sum(buckets)
    value = n_workers * grad_bytes / (ms_per_step * 1e-3) / 1e9

    # ---- end to end through the public API with host buffers
    if multi:
        host_in = [x.cpu().pin_memory() for x in grads]
        host_out = [torch.empty_like(h).pin_memory() for h in host_in]
    else:
        host_in = [[x.cpu().pin_memory() for x in ws] for ws in grads]
        host_out = [[torch.empty_like(h).pin_memory() for h in ws] for ws in host_in]

    # Bucket pipeline (what a DDP comm hook sees): bucket b's H2D on one copy
    # stream, its TAR call on the compute stream once it has landed, its D2H
    # on a second copy stream as soon as it is done -- so bucket b's D2H
    # overlaps bucket b+1's H2D (the two PCIe directions run concurrently).
    h2d_st = torch.cuda.Stream(dev)
    d2h_st = torch.cuda.Stream(dev)
    if multi:
        dev_in = [torch.empty_like(x) for x in grads]
        dev_out = [torch.empty_like(x) for x in grads]
    else:
        dev_in = [[torch.empty_like(x) for x in ws] for ws in grads]
        dev_out = [[torch.empty_like(x) for x in ws] for ws in grads]

    def e2e_step():
        gen = state["gen"]
        h2d_st.wait_stream(stream)
        d2h_st.wait_stream(stream)
        landed = []
        with torch.cuda.stream(h2d_st):
            for b in range(len(buckets)):
                if multi:
                    dev_in[b].copy_(host_in[b], non_blocking=True)
                else:
                    for d, h in zip(dev_in[b], host_in[b]):
                        d.copy_(h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d_st)
                landed.append(ev)
        for b in range(len(buckets)):
            stream.wait_event(landed[b])
            call_bucket(b, gen, dev_in, dev_out, False)
            done = torch.cuda.Event()
            done.record(stream)
            d2h_st.wait_event(done)
            with torch.cuda.stream(d2h_st):
                if multi:
                    host_out[b].copy_(dev_out[b], non_blocking=True)
                else:
                    for h, d in zip(host_out[b], dev_out[b]):
                        h.copy_(d, non_blocking=True)
        stream.wait_stream(d2h_st)
        state["gen"] += 1

    e2e_step()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        e2e_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(ev0.elapsed_time(ev1)) / e2e_steps
    per_rank_workers = 1 if multi else n_workers
    io_bytes = per_rank_workers * grad_bytes
    e2e = {"value": round(n_workers * grad_bytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
           "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": io_bytes, "d2h_bytes_per_step": io_bytes,
           "pipeline": "per bucket: H2D stream -> TAR call -> D2H stream (D2H of b overlaps H2D of b+1)"}

    # ---- roofline of the dominant kernel class: live CUDA-event durations of
    # pass (C), where every launch runs alone (buckets serialised); pass (B)'s
    # contended durations are reported beside them
    peaks = load_peaks()
    live = {k: v for k, v in per_kernel.items() if v[1] > 0}
    # multi-GPU: prep runs on a low-priority side stream beside the previous
    # call's persistent fused kernel (its event time is mostly waiting for SM
    # slots), so the dominant kernel is taken among the call-stream kernels
    crit = {k: v for k, v in live.items() if not (multi and k == "prep")} or live
    dom = max(crit, key=lambda k: crit[k][0])
    dom_ms, dom_n, dom_units = live[dom]

    def class_bytes(cls, nvlink=False, table=None):
        """Algorithmic bytes the timed launches of `cls` moved: per-worker
        bytes of each bucket x worker-passes (units spread evenly over buckets)."""
        units = (table or live)[cls][2]
        per_b = 0
        for L in buckets:
            dim = next_pow2(L) if ht else L
            if nvlink:
                # stage 1 in (+ stage 2 in for the fused kernel), per direction
                k = 2 if cls in ("fused", "small") else 1
                per_b += k * 4 * dim * (n_workers - 1) // n_workers
            else:
                per_b += kernel_bytes(cls, dim, L, n_workers, s_in, s_out)
        return units * per_b / len(buckets)

    achieved = class_bytes(dom) / (dom_ms * 1e-3) / 1e9
    if multi and dom in ("aggregate", "dec_first", "fused", "small"):
        nv_ach = class_bytes(dom, nvlink=True) / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "nvlink", "achieved": round(nv_ach, 1), "peak": nvlink_peak(n_workers), "unit": "GB/s",
                "frac": round(nv_ach / nvlink_peak(n_workers), 4), "kernel": dom,
                "peak_src": "measured all-peer SM pull" if n_workers in NVLINK_ALLPEER_GBS else "measured single-peer pull",
                "hbm_achieved": round(achieved, 1), "traffic": None}
    else:
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4), "kernel": dom, "peak_src": peaks["src"],
                "traffic": None}
    roof["timing"] = ("live CUDA events around every launch, timed pass (C): K steps with the buckets "
                      "serialised (each launch alone on the GPU)")
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    tr = ncu_traffic(dom, multi)
    if tr is not None:
        roof["traffic"], roof["traffic_src"] = tr[0], tr[1] + " (cold-cache ncu replay, one launch)"

    def table(per):
        lv = {k: v for k, v in per.items() if v[1] > 0}
        return {k: {"ms_per_step": round(v[0] / args.steps, 4), "launches_per_step": v[1] / args.steps,
                    "avg_launch_us": round(v[0] / v[1] * 1e3, 2),
                    "hbm_gbs": round(class_bytes(k, table=lv) / (v[0] * 1e-3) / 1e9, 1)}
                for k, v in lv.items()}

    kernels = table(per_kernel)
    kernels_contended = table(per_contended)

    # whole-step roofline: max(HBM_alg/HBM, NVL/NVLink)
    hbm_alg, nvl = step_alg_bytes(buckets, n_workers, s_in, s_out, ht)
    hbm_alg *= per_rank_workers
    t_roof = max(hbm_alg / (peaks["hbm_gbs"] * 1e9), (nvl / (nvlink_peak(n_workers) * 1e9)) if multi else 0.0)
    step_roof = {"t_roof_ms": round(t_roof * 1e3, 4), "frac": round(t_roof * 1e3 / ms_per_step, 4),
                 "hbm_alg_bytes": hbm_alg, "nvlink_bytes_per_dir": nvl if multi else 0}

    out = {
        "metric": "bucket allreduce GB/s (TAR+RHT)",
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if dt_name == "f32" else "bf16->f32",
        "data": "synthetic (torch.randn gradients)",
        "config": {"workload": args.workload, "desc": desc, "buckets": len(buckets),
                   "bucket_entries": per, "total_entries": total, "workers": n_workers,
                   "workers_per_gpu": per_rank_workers, "ht": args.ht, "drop": drop,
                   "mask": "datagram coin, 350-entry packets" if drop > 0 else "lossless",
                   "parallelism": f"tar{n_workers}", "l2": "inputs larger than L2 (no flush)",
                   "value_def": "aggregate over all workers: workers x gradient bytes / step time "
                                "(= n x the per-worker algBW s_in*L/t of SURVEY 8(d))",
                   "timed_passes": "(A) value / ms_per_step: buckets pipelined, two in flight; "
                                   "(B) the same with per-launch events -> kernels_contended; "
                                   "(C) buckets serialised with per-launch events -> kernels, roofline"},
        "algbw_per_worker_gbs": round(grad_bytes / (ms_per_step * 1e-3) / 1e9, 3),
        "ms_per_step_serialized": round(ms_serial, 4),
        "ms_per_step_with_kernel_events": round(ms_events, 4),
        "e2e": e2e,
        "roofline": roof,
        "step_roofline": step_roof,
        "kernels": kernels,
        "kernels_contended": kernels_contended,
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and not multi and not args.no_cpu_baseline:
        ncores = len(os.sched_getaffinity(0))
        thr = min(n_workers, ncores)
        # bounded sample of the same workload: its buckets in order until >= 10 s of
        # CPU work (ResNet-50: the whole 4-bucket step, ~10 s), at most ~30 s
        done_b, done_bytes, secs = 0, 0, 0.0
        for L in buckets:
            _, dt = cpu_baseline(L, n_workers, drop, ht, thr)
            done_b += 1
            done_bytes += n_workers * s_in * L
            secs += dt
            if secs >= 10.0 or secs + dt > 30.0:
                break
        gbs = done_bytes / secs / 1e9
        out["cpu_baseline"] = {"value": round(gbs, 6), "unit": "GB/s", "cores": thr, "kind": "port",
                               "sample": f"{done_b} of {len(buckets)} buckets of the step x {n_workers} workers, "
                                         f"oracle port (numpy, fp64), {secs:.1f}s, {ncores} cores visible"}
    if not multi and args.workload != "headline":
        out["headline"] = headline_line(args, dev, stream)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if multi:
        import torch.distributed as dist

        comm.close()
        dist.destroy_process_group()


def headline_line(args, dev, stream) -> dict:
    """The north-star bucket (25,000,000 fp32 entries, D = 2^25) at N=1 with
    the same co-resident workers and drop model, timed like pass (A): K
    generations, device time, the whole-step roofline of SURVEY 8(d)."""
    import torch

    from paper_2310_06993_b200.collectives import MaskSpec, local_join, tar_allreduce_local

    L, n = WORKLOADS["headline"][0], args.workers
    g = torch.Generator(device=dev).manual_seed(4321)
    xs = [torch.randn(L, device=dev, generator=g) for _ in range(n)]
    outs = [torch.empty_like(x) for x in xs]

    def step(gen):
        masks = MaskSpec.coin(7919 * gen + 1, args.drop) if args.drop > 0 else MaskSpec.none()
        tar_allreduce_local(xs, rotation=gen % n, ht=True, job_seed=7, generation=gen, bucket_id=0, masks=masks,
                            out=outs, async_op=True)
        local_join()

    for gen in range(args.warmup):
        step(gen)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for gen in range(args.steps):
        step(args.warmup + gen)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    hbm_alg, _nvl = step_alg_bytes([L], n, 4, 4, True)
    hbm_alg *= n
    t_roof = hbm_alg / (load_peaks()["hbm_gbs"] * 1e9)
    del xs, outs
    return {"workload": "headline", "desc": WORKLOADS["headline"][3], "workers": n, "steps": args.steps,
            "ms_per_step": round(ms, 4), "value": round(n * 4 * L / (ms * 1e-3) / 1e9, 3), "unit": "GB/s",
            "step_roofline": {"t_roof_ms": round(t_roof * 1e3, 4), "frac": round(t_roof * 1e3 / ms, 4),
                              "hbm_alg_bytes": hbm_alg}}


# ------------------------------------------------------------ reference arm
REF_BUDGET_S = 180.0  # the reference arm's timed steps end within a few minutes


def run_reference(args):
    """The reference's CPU algorithm -- the oracle port of ubar (numpy fp64,
    /root/reference is not on the GPU box): rht_encode x n, _mean_received per
    owner, assembly, rht_decode x n under the same datagram-coin masks, on the
    same buckets as our arm (a step = every bucket of the workload, same
    metric).  Rank 0 only; the other ranks exit."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    total, per, dt_name, desc = WORKLOADS[args.workload]
    buckets = bucket_sizes(total, per)
    n_workers = world if world > 1 else args.workers
    ht = args.ht == "on"
    ncores = len(os.sched_getaffinity(0))
    thr = min(n_workers, ncores)
    # warm-up steps on a 1/16 sample of the first bucket (numpy / allocator
    # paths warm; the timed steps run the full buckets)
    for _ in range(args.warmup):
        cpu_baseline(max(1, buckets[0] // 16), n_workers, args.drop, ht, thr)
    # Bounded: a step is every bucket of the workload unless K such steps
    # would take longer than REF_BUDGET_S; then every step is the first nb
    # buckets (a bounded sample of the same workload, same metric: bytes / s).
    t0 = cpu_baseline(buckets[0], n_workers, args.drop, ht, thr)[1]
    nb = len(buckets)
    if args.steps * t0 * len(buckets) > REF_BUDGET_S:
        nb = max(1, min(len(buckets), int(REF_BUDGET_S / (args.steps * t0))))
    secs = []
    for k in range(args.steps):
        secs.append((t0 if k == 0 else cpu_baseline(buckets[0], n_workers, args.drop, ht, thr)[1])
                    + sum(cpu_baseline(L, n_workers, args.drop, ht, thr)[1] for L in buckets[1:nb]))
    t = sum(secs) / len(secs)
    s_in = 2 if dt_name == "bf16" else 4
    val = n_workers * s_in * sum(buckets[:nb]) / t / 1e9
    out = {
        "metric": "bucket allreduce GB/s (TAR+RHT)", "value": round(val, 6), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": args.workload, "desc": desc, "buckets": len(buckets), "bucket_entries": per,
                   "total_entries": total, "workers": n_workers, "ht": args.ht, "drop": args.drop,
                   "same_config": nb == len(buckets), "buckets_per_timed_step": nb,
                   "value_def": "aggregate over all workers: workers x gradient bytes / step time"},
        "cpu_baseline": {"value": round(val, 6), "unit": "GB/s", "cores": thr, "kind": "port",
                         "sample": f"{nb} of the workload's {len(buckets)} buckets (up to {per} entries) x "
                                   f"{n_workers} workers per step (oracle port of ubar: numpy fp64, threads over "
                                   f"workers; all buckets unless K steps would exceed {REF_BUDGET_S:.0f} s); "
                                   f"warm-up on a 1/16 sample"},
        "e2e": {"value": round(val, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=sorted(WORKLOADS))
    ap.add_argument("--workers", type=int, default=4, help="co-resident workers at --gpus 1")
    ap.add_argument("--drop", type=float, default=0.01)
    ap.add_argument("--ht", default="on", choices=["on", "off"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
