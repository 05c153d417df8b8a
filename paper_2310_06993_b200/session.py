"""Generation-by-generation driver of the GPU hot path.

Mirrors the hot-path contract of ``SimSession.run_generation``
(``/root/reference/pkg/src/ubar/runner.py:211-276``): HT gating (:217,
:202-209 for on/off), the per-generation RHT seed
``derive_seed(seed, g % 65536, g)`` (:219-222), encode -> TAR -> decode with
EmptyReception -> zeros (:248-258), and ``generation += 1``,
``rotation = (r + 1) % n`` (:274-275).  The simulated network is replaced by
seeded drop masks; calibration, controllers and safeguards are out of scope
 -- the received counts a report carries are what they consume.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .collectives import MaskSpec, expected_counts, tar_allreduce_local
from .hadamard import derive_seed, next_pow2

_COIN_TAG = 0x636F696E  # "coin": per-generation coin seeds


@dataclass
class GenerationReport:
    """Subset of runner.py:43-60 the hot path produces."""

    generation: int
    rotation: int
    ht_used: bool
    results: list
    received: object  # CUDA int64 [2, n] received entries per (stage, dst)
    expected: np.ndarray  # [2, n]

    @property
    def loss_rates(self) -> np.ndarray:
        """Per node 1 - received/expected over both stages (NodeStats.loss_rate
        semantics, simdriver.py:328-333)."""
        got = self.received.cpu().numpy().sum(axis=0)
        exp = self.expected.sum(axis=0)
        return np.where(exp > 0, 1.0 - got / np.maximum(exp, 1), 0.0)

    @property
    def max_loss(self) -> float:
        return float(self.loss_rates.max())


class GpuSession:
    """n workers co-resident on one GPU.

    masks: "none" | "coin" | a callable ``(generation, rotation, dim) -> MaskSpec``.
    With "coin", generation g uses coin seed ``derive_seed(seed, 'coin', g)``
    and ``drop_prob``, packets of ``max_payload`` bytes.
    """

    def __init__(self, n: int, seed: int, ht: str = "on", drop_prob: float = 0.0,
                 max_payload: int = 1400, masks="coin"):
        if ht not in ("on", "off"):
            raise ValueError(f"unknown ht mode {ht!r} (auto needs the UBT controllers, out of scope)")
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

    def ht_active(self) -> bool:
        return self.ht_mode == "on"

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
        self.generation += 1
        self.rotation = (self.rotation + 1) % self.n
        return rep
