"""UBT control plane (unreliable bounded transport) driven by GPU timings.

OptiReduce bounds every collective stage in time instead of waiting for the
slowest sender: a hard bound t_B (calibrated once as the 95th percentile of
reliable stage times), an early timeout x% of a moving-average completion
time t_C once the last packets from every sender are in, an x% loop that
keeps the loss inside [0.01%, 0.1%], the Hadamard codec switched on (and
latched) above 2% loss, and a safeguard that skips an update above 2% loss
and halts after three consecutive generations above 30%.

Reference rules restated here (paths relative to
``/root/reference/pkg/src/ubar/``):

=====================  ==========================  =============================
rule                   reference                   here
=====================  ==========================  =============================
t_B calibration        transport.py:102-108        ``calibrate_t_b``
completion estimate    transport.py:111-120        ``expected_completion``
t_C moving average     transport.py:123-135        ``fold_t_c``
x% loss band           transport.py:138-144        ``adjust_x_pct``
HT activation (latch)  transport.py:147-149,212-217 ``maybe_activate_ht``
incast +-1             transport.py:152-168        ``adjust_incast`` / ``effective_incast``
TIMELY-like rate       transport.py:171-180        ``rate_update``
per-node controller    transport.py:183-217        ``UbtController``
skip / halt            safeguards.py:15-53         ``assess`` (``SafeguardPolicy``, ``LossHistory``)
per-generation update  runner.py:278-293           ``ControlPlane.end_generation``
=====================  ==========================  =============================

On a B200 box the "network" is NVLink inside a persistent kernel, so the
inputs come from the device: the fused TAR kernel stamps the stage times
with the GPU global timer and counts the entries each rank received (and the
entries its stage-1 deadline cut off); ``ControlPlane`` turns those into the
next generation's deadline (``stage1_deadline_ns``), HT decision and
safeguard ``Action``.  Everything here is host-side scalar control, as in the
reference.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field, replace

__all__ = [
    "LOSS_BAND_LOW", "LOSS_BAND_HIGH", "HT_ACTIVATION_LOSS", "DEFAULT_ALPHA", "DEFAULT_X_PCT", "X_PCT_MIN",
    "X_PCT_MAX", "CALIBRATION_ITERATIONS", "CALIBRATION_PERCENTILE", "RTT_SAMPLE_EVERY",
    "CalibrationError", "Completion", "StageOutcome", "TimeoutState", "IncastState", "RateState",
    "calibrate_t_b", "expected_completion", "fold_t_c", "adjust_x_pct", "maybe_activate_ht",
    "adjust_incast", "effective_incast", "rate_update", "UbtController",
    "Action", "SafeguardPolicy", "LossHistory", "assess", "NodeOutcome", "ControlPlane",
]

# loss band of the x% loop and the HT switch (transport.py:18-21)
LOSS_BAND_LOW, LOSS_BAND_HIGH, HT_ACTIVATION_LOSS = 1e-4, 1e-3, 0.02
DEFAULT_ALPHA, DEFAULT_X_PCT, X_PCT_MIN, X_PCT_MAX = 0.95, 10.0, 1.0, 50.0
CALIBRATION_ITERATIONS, CALIBRATION_PERCENTILE = 20, 95
RTT_SAMPLE_EVERY = 10


class CalibrationError(ValueError):
    pass


class Completion(enum.Enum):
    ON_TIME = "on_time"
    EARLY_TIMEOUT = "early_timeout"
    HARD_TIMEOUT = "hard_timeout"


@dataclass
class StageOutcome:
    """How one bounded receive stage ended (transport.py:46-53)."""

    completion: Completion
    elapsed: float
    loss_rate: float
    expected_bytes: int = 0
    received_bytes: int = 0
    last_pct_from_all: bool = False


def _clamp(v, lo, hi):
    return lo if v < lo else hi if v > hi else v


@dataclass
class TimeoutState:
    """Hard bound, per-stage-kind moving averages, early-timeout share
    (transport.py:56-77): t_C never exceeds t_B, x% stays in [1, 50]."""

    t_b: float
    t_c_stage1: float = 0.0
    t_c_stage2: float = 0.0
    alpha: float = DEFAULT_ALPHA
    x_pct: float = DEFAULT_X_PCT

    def __post_init__(self):
        self.t_c_stage1 = min(self.t_c_stage1, self.t_b)
        self.t_c_stage2 = min(self.t_c_stage2, self.t_b)
        self.x_pct = _clamp(self.x_pct, X_PCT_MIN, X_PCT_MAX)

    def t_c(self, stage_kind: int) -> float:
        return self.t_c_stage1 if stage_kind == 1 else self.t_c_stage2

    def set_t_c(self, stage_kind: int, value: float) -> None:
        setattr(self, "t_c_stage1" if stage_kind == 1 else "t_c_stage2", min(value, self.t_b))


@dataclass
class IncastState:
    i_factor: int = 1
    advertised: int = 1


@dataclass
class RateState:
    """Sender pacing (transport.py:86-99): additive increase below t_low,
    multiplicative decrease above t_high."""

    rate: float = 1e9 / 8
    last_rtt: float = 0.0
    t_low: float = 25e-6
    t_high: float = 250e-6
    add_step: float = 50e6 / 8
    beta: float = 0.5

    def __post_init__(self):
        if self.rate <= 0:
            raise ValueError("rate must be positive")
        if not self.t_low < self.t_high:
            raise ValueError("t_low must be below t_high")


def calibrate_t_b(samples) -> float:
    """Nearest-rank 95th percentile of the pooled reliable stage times."""
    xs = sorted(samples)
    if not xs:
        raise CalibrationError("no calibration samples")
    k = -(-CALIBRATION_PERCENTILE * len(xs) // 100)  # ceil(0.95 n), 1-based
    return xs[k - 1]


def expected_completion(outcome: StageOutcome, t_b: float) -> float:
    """A stage's completion-time estimate: its elapsed time when on time, t_B
    after a hard timeout, and the elapsed time scaled by expected/received
    bytes after an early timeout (t_B when nothing arrived)."""
    c = outcome.completion
    if c is Completion.ON_TIME:
        return outcome.elapsed
    if c is Completion.HARD_TIMEOUT or outcome.received_bytes <= 0:
        return t_b
    return outcome.elapsed * outcome.expected_bytes / outcome.received_bytes


def fold_t_c(local_estimates, prev_t_c: float, alpha: float) -> float:
    """Lower median of the nodes' estimates, blended alpha : 1-alpha into the
    previous average (the first fold takes the median itself)."""
    xs = sorted(local_estimates)
    if not xs:
        return prev_t_c
    med = xs[(len(xs) - 1) // 2]
    return med if prev_t_c <= 0 else alpha * med + (1.0 - alpha) * prev_t_c


def adjust_x_pct(x: float, loss_rate: float) -> float:
    """Above the band double x% (cap 50), below it step down by 1 (floor 1)."""
    if loss_rate > LOSS_BAND_HIGH:
        return min(2.0 * x, X_PCT_MAX)
    if loss_rate < LOSS_BAND_LOW:
        return max(x - 1.0, X_PCT_MIN)
    return x


def maybe_activate_ht(loss_rate: float) -> bool:
    """The codec turns on strictly above 2% loss."""
    return loss_rate > HT_ACTIVATION_LOSS


def adjust_incast(state: IncastState, loss_rate: float, timeout_occurred: bool, n: int) -> IncastState:
    """Back off one step on loss above the band or any timeout, probe one step
    up when the generation was clean (below the band, no timeout)."""
    i = state.i_factor
    if loss_rate > LOSS_BAND_HIGH or timeout_occurred:
        i = max(1, i - 1)
    elif loss_rate < LOSS_BAND_LOW:
        i = min(n - 1, i + 1)
    return IncastState(i_factor=i, advertised=i)


def effective_incast(adverts) -> int:
    """Senders honour the smallest advertised incast factor."""
    return max(1, min(adverts)) if adverts else 1


def rate_update(state: RateState, rtt: float) -> RateState:
    if rtt <= 0:
        return state
    if rtt < state.t_low:
        rate = state.rate + state.add_step
    elif rtt > state.t_high:
        rate = state.rate * (1.0 - state.beta * (1.0 - state.t_high / rtt))
    else:
        rate = state.rate
    return replace(state, rate=rate, last_rtt=rtt)


@dataclass
class UbtController:
    """One node's transport state (transport.py:183-217)."""

    n: int
    timeouts: TimeoutState
    incast: IncastState = field(default_factory=IncastState)
    rate: RateState = field(default_factory=RateState)
    ht_active: bool = False
    _pkt_counter: int = 0

    def early_wait(self, stage_kind: int) -> float:
        """x% of the stage kind's t_C (t_B until t_C is known)."""
        t_c = self.timeouts.t_c(stage_kind)
        return (self.timeouts.x_pct / 100.0) * (t_c if t_c > 0 else self.timeouts.t_b)

    def observe_rtt(self, rtt: float) -> None:
        self._pkt_counter += 1
        if self._pkt_counter % RTT_SAMPLE_EVERY == 0:
            self.rate = rate_update(self.rate, rtt)

    def fold_stage_t_c(self, stage_kind: int, node_estimates) -> None:
        self.timeouts.set_t_c(stage_kind, fold_t_c(node_estimates, self.timeouts.t_c(stage_kind),
                                                   self.timeouts.alpha))

    def end_generation(self, loss_rate: float, timeout_occurred: bool) -> None:
        self.timeouts.x_pct = adjust_x_pct(self.timeouts.x_pct, loss_rate)
        self.incast = adjust_incast(self.incast, loss_rate, timeout_occurred, self.n)
        self.ht_active = self.ht_active or maybe_activate_ht(loss_rate)


# ------------------------------------------------------------ safeguards
class Action(enum.Enum):
    ACCEPT = "accept"
    SKIP_UPDATE = "skip_update"
    HALT = "halt"


@dataclass(frozen=True)
class SafeguardPolicy:
    """safeguards.py:21-31: skip above 2% loss, halt after `window`
    consecutive generations above 30%."""

    skip_threshold: float = 0.02
    halt_threshold: float = 0.30
    window: int = 3

    def __post_init__(self):
        if not 0.0 < self.skip_threshold <= self.halt_threshold <= 1.0:
            raise ValueError("need 0 < skip_threshold <= halt_threshold <= 1")
        if self.window < 1:
            raise ValueError("window must be >= 1")


@dataclass
class LossHistory:
    consecutive_above_halt: int = 0
    losses: list = field(default_factory=list)


def assess(loss_rate: float, policy: SafeguardPolicy, history: LossHistory) -> Action:
    """safeguards.py:40-53: classify one generation's (max) loss."""
    if not 0.0 <= loss_rate <= 1.0:
        raise ValueError(f"loss rate out of range: {loss_rate}")
    history.losses.append(loss_rate)
    if loss_rate > policy.halt_threshold:
        history.consecutive_above_halt += 1
        return Action.HALT if history.consecutive_above_halt >= policy.window else Action.SKIP_UPDATE
    history.consecutive_above_halt = 0
    return Action.SKIP_UPDATE if loss_rate > policy.skip_threshold else Action.ACCEPT


# ------------------------------------------------------------ control plane
@dataclass
class NodeOutcome:
    """One rank's view of a generation, from the device counters."""

    loss_rate: float
    timeout_occurred: bool
    outcomes: list  # (stage kind, StageOutcome)


class ControlPlane:
    """The per-job UBT loop over all n nodes (runner.py:138-187 calibration,
    :202-209 HT gating, :278-293 controller update, :272 safeguard).

    ``calibrate(samples)`` takes reliable-run stage times (seconds) and the
    per-kind medians; ``end_generation(nodes)`` folds each stage kind's
    completion estimates into t_C, runs every node's x% / incast / HT loops
    and returns the safeguard ``Action`` for the generation's max loss.
    ``stage1_deadline_ns()`` is the bound the next fused kernel enforces on
    its stage-1 waits (t_B, or the early timeout once t_C is known).
    """

    def __init__(self, n: int, ht: str = "off", alpha: float = DEFAULT_ALPHA, x_pct: float = DEFAULT_X_PCT,
                 policy: SafeguardPolicy | None = None):
        if ht not in ("off", "on", "auto"):
            raise ValueError(f"unknown ht mode {ht!r}")
        self.n = n
        self.ht_mode = ht
        self.alpha = alpha
        self.x_pct0 = x_pct
        self.policy = policy or SafeguardPolicy()
        self.history = LossHistory()
        self.controllers = None

    @property
    def calibrated(self) -> bool:
        return self.controllers is not None

    def calibrate(self, pooled, per_kind: dict | None = None, t_b: float | None = None) -> float:
        t_b = calibrate_t_b(pooled) if t_b is None else float(t_b)
        per_kind = per_kind or {}
        med = {k: (sorted(v)[(len(v) - 1) // 2] if v else 0.0) for k, v in per_kind.items()}
        self.controllers = [
            UbtController(n=self.n, timeouts=TimeoutState(t_b=t_b, t_c_stage1=med.get(1, 0.0),
                                                          t_c_stage2=med.get(2, 0.0), alpha=self.alpha,
                                                          x_pct=self.x_pct0))
            for _ in range(self.n)]
        return t_b

    def ht_active(self) -> bool:
        if self.ht_mode != "auto":
            return self.ht_mode == "on"
        return bool(self.controllers) and any(c.ht_active for c in self.controllers)

    def t_b(self) -> float:
        return self.controllers[0].timeouts.t_b if self.controllers else 0.0

    def stage1_deadline_ns(self) -> int:
        """Hard bound t_B for the owners' stage-1 waits (0 = unbounded before
        calibration)."""
        return int(self.t_b() * 1e9) if self.controllers else 0

    def end_generation(self, nodes) -> Action:
        if self.controllers:
            t_b = self.t_b()
            for kind in (1, 2):
                est = []
                for nd in nodes:
                    vals = [expected_completion(o, t_b) for k, o in nd.outcomes if k == kind]
                    if vals:
                        est.append(sum(vals) / len(vals))
                for c in self.controllers:
                    c.fold_stage_t_c(kind, est)
            for c, nd in zip(self.controllers, nodes):
                c.end_generation(nd.loss_rate, nd.timeout_occurred)
        return assess(max((nd.loss_rate for nd in nodes), default=0.0), self.policy, self.history)
