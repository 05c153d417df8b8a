"""Generation-by-generation drivers of the GPU hot path.

Both mirror the hot-path contract of ``SimSession.run_generation``
(``/root/reference/pkg/src/ubar/runner.py:211-276``): HT gating (:217,
:202-209 on / off / auto-latched), the per-generation RHT seed
``derive_seed(seed, g % 65536, g)`` (:219-222), encode -> TAR -> decode with
EmptyReception -> zeros (:248-258), the controller update (:278-293), the
safeguard action (:272) and ``generation += 1``, ``rotation = (r + 1) % n``
(:274-275).

* ``GpuSession``: n workers co-resident on one GPU (the SimSession shape);
  the lossy network is the seeded drop masks; the UBT loops run on the
  received counts (x%, incast, HT latch, skip / halt).  One GPU has no
  transport delay, so t_B / t_C stay at their override / calibration.
* ``BoundedSession``: one rank per GPU over NVLink (``TarCommunicator``);
  stage 1 is bounded in time on the device (``optr_tar_bounded``): t_B is
  calibrated from the fused kernel's own stage times over reliable
  generations (runner.py:138-187) and every later generation's owners stop
  waiting for a late peer at t_B, counting its entries as lost.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import ubt
from .collectives import MaskSpec, expected_counts, tar_allreduce_local
from .hadamard import derive_seed, next_pow2

_COIN_TAG = 0x636F696E  # "coin": per-generation coin seeds


@dataclass
class GenerationReport:
    """The runner's report (runner.py:43-60) for the hot path."""

    generation: int
    rotation: int
    ht_used: bool
    results: list
    received: object  # CUDA int64 [2, n] (GpuSession) / host [2, n] (BoundedSession) received entries
    expected: np.ndarray  # [2, n]
    action: ubt.Action = ubt.Action.ACCEPT
    stage_times: object = None  # BoundedSession: [n, 2] seconds (stage 1, stage 2) per rank
    cut: object = None  # BoundedSession: [n] stage-1 entries cut by the deadline per rank

    @property
    def loss_rates(self) -> np.ndarray:
        """Per node 1 - received/expected over both stages (NodeStats.loss_rate,
        simdriver.py:32-36)."""
        got = np.asarray(self.received.cpu().numpy() if hasattr(self.received, "cpu") else self.received).sum(axis=0)
        exp = self.expected.sum(axis=0)
        return np.where(exp > 0, 1.0 - got / np.maximum(exp, 1), 0.0)

    @property
    def max_loss(self) -> float:
        return float(self.loss_rates.max())

    @property
    def mean_loss(self) -> float:
        return float(self.loss_rates.mean())


class GpuSession:
    """n workers co-resident on one GPU.

    masks: "none" | "coin" | a callable ``(generation, rotation, dim) -> MaskSpec``.
    With "coin", generation g uses coin seed ``derive_seed(seed, 'coin', g)``
    and ``drop_prob``, packets of ``max_payload`` bytes.  ``ht``: "on" /
    "off" / "auto" (latched on once any node's loss exceeds 2%,
    transport.py:147-149,212-217).
    """

    def __init__(self, n: int, seed: int, ht: str = "on", drop_prob: float = 0.0,
                 max_payload: int = 1400, masks="coin", policy: ubt.SafeguardPolicy | None = None,
                 t_b: float = 1.0):
        if ht not in ("on", "off", "auto"):
            raise ValueError(f"unknown ht mode {ht!r}")
        if n < 2:
            raise ValueError("need at least 2 nodes")
        self.n = n
        self.seed = int(seed)
        self.ht_mode = ht
        self.drop_prob = float(drop_prob)
        self.max_payload = int(max_payload)
        self.masks = masks
        self.rotation = 0
        self.generation = 0
        self.control = ubt.ControlPlane(n, ht=ht, policy=policy)
        self.control.calibrate([], t_b=t_b)

    def ht_active(self) -> bool:
        return self.control.ht_active()

    def mask_spec(self, dim: int) -> MaskSpec:
        if callable(self.masks):
            return self.masks(self.generation, self.rotation, dim)
        if self.masks == "none" or self.drop_prob == 0.0:
            return MaskSpec.none(self.max_payload)
        coin_seed = derive_seed(self.seed, _COIN_TAG, self.generation)
        return MaskSpec.coin(coin_seed, self.drop_prob, self.max_payload)

    def run_generation(self, buckets: list, out_dtype=None, stream=None) -> GenerationReport:
        bucket_len = len(buckets[0])
        ht_used = self.ht_active()
        dim = next_pow2(bucket_len) if ht_used else bucket_len
        spec = self.mask_spec(dim)
        outs, counts, _ = tar_allreduce_local(
            buckets, rotation=self.rotation, ht=ht_used, job_seed=self.seed,
            generation=self.generation, masks=spec, out_dtype=out_dtype, stream=stream)
        rep = GenerationReport(self.generation, self.rotation, ht_used, outs, counts,
                               expected_counts(dim, self.n, self.rotation))
        loss = rep.loss_rates
        rep.action = self.control.end_generation(
            [ubt.NodeOutcome(loss_rate=float(lr), timeout_occurred=False, outcomes=[]) for lr in loss])
        self.generation += 1
        self.rotation = (self.rotation + 1) % self.n
        return rep


class BoundedSession:
    """One rank's OptiReduce loop over NVLink (one process per GPU).

    ``transport="ubt"``: before the first lossy generation,
    ``calibration_iterations`` reliable generations (no drops, no deadline)
    time the fused kernel's stages on every rank; t_B = nearest-rank p95 of
    the pooled stage times (transport.py:102-108), t_C seeds from the
    per-stage medians.  Each generation then runs with stage 1 bounded at
    t_B on the device and feeds the ranks' losses, cut-offs and stage times
    to the controllers; the report carries the safeguard action.
    ``transport="reliable"``: no deadline, no calibration.
    """

    def __init__(self, comm, seed: int, ht: str = "auto", drop_prob: float = 0.0, max_payload: int = 1400,
                 transport: str = "ubt", calibration_iterations: int = ubt.CALIBRATION_ITERATIONS,
                 t_b: float | None = None, alpha: float = ubt.DEFAULT_ALPHA, x_pct: float = ubt.DEFAULT_X_PCT,
                 policy: ubt.SafeguardPolicy | None = None):
        if transport not in ("ubt", "reliable"):
            raise ValueError(f"unknown transport {transport!r}")
        self.comm = comm
        self.n = comm.world
        self.rank = comm.rank
        self.seed = int(seed)
        self.drop_prob = float(drop_prob)
        self.max_payload = int(max_payload)
        self.transport = transport
        self.calibration_iterations = int(calibration_iterations)
        self.t_b_override = t_b
        self.control = ubt.ControlPlane(self.n, ht=ht, alpha=alpha, x_pct=x_pct, policy=policy)
        self.rotation = 0
        self.generation = 0

    def _gather(self, t):
        """all_gather of a small int64 CUDA tensor over the communicator's group."""
        import torch
        import torch.distributed as dist

        parts = [torch.empty_like(t) for _ in range(self.n)]
        if dist.get_backend(self.comm.group) == "gloo":
            h = t.cpu()
            hp = [torch.empty_like(h) for _ in range(self.n)]
            dist.all_gather(hp, h, group=self.comm.group)
            return torch.stack(hp)
        dist.all_gather(parts, t, group=self.comm.group)
        return torch.stack(parts).cpu()

    def _call(self, x, out, ht, masks, deadline_ns, generation, rotation):
        import torch

        stats = torch.zeros(7, dtype=torch.int64, device=x.device)
        self.comm.allreduce(x, out, rotation=rotation, ht=ht, job_seed=self.seed, generation=generation,
                            masks=masks, deadline_ns=deadline_ns, stats=stats)
        return self._gather(stats)  # [n, 7]

    @staticmethod
    def _times(all_stats):
        s = all_stats.numpy().astype(np.int64)
        t1 = (s[:, 5] - s[:, 4]).clip(min=0) / 1e9
        t2 = (s[:, 6] - s[:, 4]).clip(min=0) / 1e9
        return np.stack([t1, t2], axis=1)

    def ensure_calibrated(self, bucket) -> None:
        """runner.py:138-187 on device timings: reliable generations of random
        buckets of the same length, stage times pooled over every rank."""
        import torch

        if self.control.calibrated or self.transport != "ubt":
            return
        if self.t_b_override is not None:
            self.control.calibrate([], t_b=self.t_b_override)
            return
        g = torch.Generator(device=bucket.device).manual_seed(self.seed * 1009 + self.rank)
        pooled, per_kind = [], {1: [], 2: []}
        out = torch.empty_like(bucket)
        for it in range(self.calibration_iterations):
            x = torch.randn(len(bucket), device=bucket.device, generator=g).to(bucket.dtype)
            st = self._call(x, out, True, MaskSpec.none(self.max_payload), 0, 0x7FFFFFFF - it, it % self.n)
            times = self._times(st)
            pooled += list(times.reshape(-1))
            per_kind[1] += list(times[:, 0])
            per_kind[2] += list(times[:, 1])
        self.control.calibrate(pooled, per_kind)

    def mask_spec(self) -> MaskSpec:
        if self.drop_prob == 0.0:
            return MaskSpec.none(self.max_payload)
        return MaskSpec.coin(derive_seed(self.seed, _COIN_TAG, self.generation), self.drop_prob, self.max_payload)

    def run_generation(self, bucket, out=None) -> GenerationReport:
        import torch

        self.ensure_calibrated(bucket)
        L = len(bucket)
        ht_used = self.control.ht_active()
        dim = next_pow2(L) if ht_used else L
        out = out if out is not None else torch.empty_like(bucket)
        deadline = self.control.stage1_deadline_ns() if self.transport == "ubt" else 0
        st = self._call(bucket, out, ht_used, self.mask_spec(), deadline, self.generation, self.rotation)
        s = st.numpy().astype(np.int64)
        exp = expected_counts(dim, self.n, self.rotation)
        times = self._times(st)
        nodes = []
        for q in range(self.n):
            o1 = ubt.StageOutcome(ubt.Completion.HARD_TIMEOUT if s[q, 2] > 0 else ubt.Completion.ON_TIME,
                                  float(times[q, 0]), 1.0 - s[q, 0] / max(exp[0, q], 1), int(exp[0, q]) * 4,
                                  int(s[q, 0]) * 4)
            o2 = ubt.StageOutcome(ubt.Completion.ON_TIME, float(times[q, 1]), 1.0 - s[q, 1] / max(exp[1, q], 1),
                                  int(exp[1, q]) * 4, int(s[q, 1]) * 4)
            loss = 1.0 - (s[q, 0] + s[q, 1]) / max(exp[0, q] + exp[1, q], 1)
            nodes.append(ubt.NodeOutcome(loss_rate=float(loss), timeout_occurred=bool(s[q, 2] > 0),
                                         outcomes=[(1, o1), (2, o2)]))
        rep = GenerationReport(self.generation, self.rotation, ht_used, [out], s[:, :2].T.copy(), exp,
                               stage_times=times, cut=s[:, 2].copy())
        rep.action = self.control.end_generation(nodes)
        self.generation += 1
        self.rotation = (self.rotation + 1) % self.n
        return rep
