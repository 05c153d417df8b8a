"""UBT control rules (paper_2310_06993_b200.ubt) -- CPU.

Two layers: the behaviour the reference's own tests pin
(test_transport.py / test_safeguards.py, restated), and a differential
check against the reference implementation itself on randomised inputs
(``reference`` marker: runs where /root/reference exists, i.e. in the build
container)."""

import os
import random
import sys

import pytest

from paper_2310_06993_b200 import ubt as U

REF = "/root/reference/pkg/src"


# ------------------------------------------------------------ restated pins
def test_calibrate_t_b_nearest_rank_p95():
    assert U.calibrate_t_b([float(i) for i in range(1, 101)]) == 95.0
    assert U.calibrate_t_b([3.0]) == 3.0
    assert U.calibrate_t_b([5.0, 1.0, 2.0]) == U.calibrate_t_b([1.0, 2.0, 5.0]) == 5.0
    with pytest.raises(U.CalibrationError):
        U.calibrate_t_b([])


def test_expected_completion_cases():
    o = U.StageOutcome(U.Completion.ON_TIME, 0.3, 0.0, 100, 100)
    assert U.expected_completion(o, 1.0) == 0.3
    o = U.StageOutcome(U.Completion.HARD_TIMEOUT, 0.9, 0.5, 100, 50)
    assert U.expected_completion(o, 1.0) == 1.0
    o = U.StageOutcome(U.Completion.EARLY_TIMEOUT, 0.4, 0.2, 100, 80)
    assert U.expected_completion(o, 1.0) == pytest.approx(0.5)
    o = U.StageOutcome(U.Completion.EARLY_TIMEOUT, 0.4, 1.0, 100, 0)
    assert U.expected_completion(o, 1.0) == 1.0


def test_fold_t_c():
    assert U.fold_t_c([1.0, 3.0, 2.0], 0.0, 0.95) == 2.0  # seeds with the median
    assert U.fold_t_c([1.0, 2.0, 3.0, 4.0], 0.0, 0.95) == 2.0  # lower median
    assert U.fold_t_c([2.0], 1.0, 0.95) == pytest.approx(0.95 * 2.0 + 0.05 * 1.0)
    assert U.fold_t_c([], 0.7, 0.95) == 0.7
    ts = U.TimeoutState(t_b=1.0, t_c_stage1=5.0)
    assert ts.t_c_stage1 == 1.0
    ts.set_t_c(2, 9.0)
    assert ts.t_c(2) == 1.0


def test_x_pct_band_and_caps():
    assert U.adjust_x_pct(10.0, 0.01) == 20.0
    assert U.adjust_x_pct(40.0, 0.01) == 50.0
    assert U.adjust_x_pct(10.0, 0.0) == 9.0
    assert U.adjust_x_pct(1.0, 0.0) == 1.0
    assert U.adjust_x_pct(10.0, 0.0005) == 10.0


def test_ht_latch_and_incast():
    assert not U.maybe_activate_ht(0.02) and U.maybe_activate_ht(0.0201)
    c = U.UbtController(n=4, timeouts=U.TimeoutState(t_b=1.0))
    c.end_generation(0.05, False)
    assert c.ht_active
    c.end_generation(0.0, False)
    assert c.ht_active  # latches
    s = U.IncastState(1, 1)
    s = U.adjust_incast(s, 0.0, False, 4)
    assert s.i_factor == 2
    s = U.adjust_incast(U.IncastState(3, 3), 0.0, False, 4)
    assert s.i_factor == 3  # bounded by n-1
    assert U.adjust_incast(U.IncastState(2, 2), 0.0, True, 4).i_factor == 1
    assert U.effective_incast([3, 1, 2]) == 1 and U.effective_incast([]) == 1


def test_rate_rules():
    s = U.RateState(rate=1e9)
    assert U.rate_update(s, 1e-6).rate == 1e9 + s.add_step
    assert U.rate_update(s, 1e-4).rate == 1e9
    assert U.rate_update(s, 500e-6).rate == pytest.approx(1e9 * (1 - 0.5 * (1 - 250 / 500)))
    assert U.rate_update(s, -1.0) is s
    c = U.UbtController(n=2, timeouts=U.TimeoutState(t_b=1.0))
    for _ in range(9):
        c.observe_rtt(1e-6)
    assert c.rate.rate == U.RateState().rate  # sampled every 10th packet
    c.observe_rtt(1e-6)
    assert c.rate.rate > U.RateState().rate


def test_safeguards():
    pol, h = U.SafeguardPolicy(), U.LossHistory()
    assert U.assess(0.0, pol, h) is U.Action.ACCEPT
    assert U.assess(0.05, pol, h) is U.Action.SKIP_UPDATE
    assert [U.assess(0.5, pol, h) for _ in range(3)] == [U.Action.SKIP_UPDATE, U.Action.SKIP_UPDATE, U.Action.HALT]
    h = U.LossHistory()
    U.assess(0.5, pol, h)
    U.assess(0.5, pol, h)
    U.assess(0.1, pol, h)  # streak resets below the halt threshold
    assert U.assess(0.5, pol, h) is U.Action.SKIP_UPDATE
    assert U.assess(0.9, U.SafeguardPolicy(window=1), U.LossHistory()) is U.Action.HALT
    with pytest.raises(ValueError):
        U.SafeguardPolicy(skip_threshold=0.5, halt_threshold=0.3)
    with pytest.raises(ValueError):
        U.assess(1.5, pol, h)


def test_control_plane_generation_loop():
    cp = U.ControlPlane(n=4, ht="auto")
    assert not cp.ht_active() and cp.stage1_deadline_ns() == 0
    t_b = cp.calibrate([1e-3 * (i + 1) for i in range(20)], {1: [2e-3, 4e-3], 2: [1e-3]})
    assert t_b == 19e-3 and cp.stage1_deadline_ns() == 19_000_000
    out = U.StageOutcome(U.Completion.ON_TIME, 3e-3, 0.0, 400, 400)
    nodes = [U.NodeOutcome(loss_rate=0.03 if i == 2 else 0.0, timeout_occurred=False, outcomes=[(1, out), (2, out)])
             for i in range(4)]
    assert cp.end_generation(nodes) is U.Action.SKIP_UPDATE  # max loss 3% > 2%
    assert cp.ht_active()  # node 2 saw > 2%: the codec latches on
    assert cp.controllers[0].timeouts.t_c_stage1 == pytest.approx(0.95 * 3e-3 + 0.05 * 2e-3)


# ------------------------------------------------------------ vs the reference
@pytest.mark.reference
@pytest.mark.skipif(not os.path.isdir(REF), reason="/root/reference not present")
def test_rules_match_reference_randomised():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    try:
        from ubar import safeguards as RS
        from ubar import transport as RT
    finally:
        sys.path.remove(REF)
    rnd = random.Random(7)
    for _ in range(300):
        xs = [rnd.random() for _ in range(rnd.randint(1, 60))]
        assert U.calibrate_t_b(xs) == RT.calibrate_t_b(xs)
        prev = rnd.choice([0.0, rnd.random()])
        assert U.fold_t_c(xs, prev, 0.95) == RT.fold_t_c(xs, prev, 0.95)
        loss = rnd.choice([0.0, 5e-5, 5e-4, 2e-3, 0.02, 0.0200001, rnd.random()])
        x = rnd.uniform(1, 50)
        assert U.adjust_x_pct(x, loss) == RT.adjust_x_pct(x, loss)
        assert U.maybe_activate_ht(loss) == RT.maybe_activate_ht(loss)
        i = rnd.randint(1, 7)
        to = rnd.random() < 0.3
        a = U.adjust_incast(U.IncastState(i, i), loss, to, 8)
        b = RT.adjust_incast(RT.IncastState(i, i), loss, to, 8)
        assert (a.i_factor, a.advertised) == (b.i_factor, b.advertised)
        rtt = rnd.choice([-1.0, 1e-6, 1e-4, 1e-3, rnd.random() * 1e-3])
        assert U.rate_update(U.RateState(rate=1e9), rtt).rate == RT.rate_update(RT.RateState(rate=1e9), rtt).rate
        comp = rnd.choice(list(U.Completion))
        e, r_ = rnd.randint(0, 1000), rnd.randint(0, 1000)
        el = rnd.random()
        ou = U.StageOutcome(comp, el, 0.0, e, r_)
        orf = RT.StageOutcome(RT.Completion(comp.value), el, 0.0, e, r_)
        assert U.expected_completion(ou, 0.7) == RT.expected_completion(orf, 0.7)
    # controllers and safeguards over random generation sequences
    for _ in range(50):
        cu = U.UbtController(n=8, timeouts=U.TimeoutState(t_b=1.0, x_pct=10.0))
        cr = RT.UbtController(n=8, timeouts=RT.TimeoutState(t_b=1.0, x_pct=10.0))
        hu, hr = U.LossHistory(), RS.LossHistory()
        pu, pr = U.SafeguardPolicy(), RS.SafeguardPolicy()
        for _g in range(30):
            loss = rnd.choice([0.0, 5e-5, 5e-4, 0.01, 0.03, 0.4])
            to = rnd.random() < 0.2
            cu.end_generation(loss, to)
            cr.end_generation(loss, to)
            assert (cu.timeouts.x_pct, cu.incast.i_factor, cu.ht_active) == \
                (cr.timeouts.x_pct, cr.incast.i_factor, cr.ht_active)
            est = [rnd.random() for _ in range(8)]
            cu.fold_stage_t_c(1, est)
            cr.fold_stage_t_c(1, est)
            assert cu.timeouts.t_c_stage1 == cr.timeouts.t_c_stage1
            assert cu.early_wait(1) == cr.early_wait(1)
            assert U.assess(loss, pu, hu).value == RS.assess(loss, pr, hr).value
