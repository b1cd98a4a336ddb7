"""F3: the paper's cost model (Eqs. 1-4) and Algorithm 1 on CPU.

Pinned to the worked examples SPEC.md derives from the paper's equations (SPEC.md:116-158
cost_model, :436-470 spec_scheduler; Eq. 2 = 0.588 s at SPEC.md:445) and to the properties
SPEC.md states (greedy-prefix optimality by exhaustive enumeration, monotone load response,
expiry safety, Eq. 4 N-independence, calibration round trip).
"""
import math
import random

import pytest

from paper_2511_20048_b200.scheduler import (CalibrationError, CostModelParams, SchedulerConfig, SpecCandidate,
                                             admitted_vs_load, calibrate, decode_overhead, expected_reduction,
                                             hybrid_batch_time, net_gain, prefill_overhead, priority_key, select_step)

P = CostModelParams()   # SPEC.md:154 defaults: d0 20 ms, gamma 0.1 ms, N0 64, alpha 0.2, 2 ms + 0.05 ms/token


def test_hybrid_batch_time_spec_examples():
    assert hybrid_batch_time((), 16, P) == pytest.approx(0.0216, abs=1e-15)
    assert hybrid_batch_time((), 0, P) == P.base_step_time
    assert hybrid_batch_time([(512, 2)], 16, P) == pytest.approx(0.0768, abs=1e-15)


def test_decode_overhead_spec_examples():
    assert decode_overhead(2, 3, 16, 8, P) == pytest.approx(0.0048, abs=1e-15)
    assert decode_overhead(0, 3, 16, 8, P) == 0.0
    # straddling the knee: N = 63, one speculative request of k = 3: 1 request below the
    # knee, 2 past it at (1 + alpha) -> 8 gamma (1 + 2 x 1.2)
    assert decode_overhead(1, 3, 63, 8, P) == pytest.approx(8 * 1e-4 * 3.4, abs=1e-15)


def test_prefill_overhead_spec_examples():
    assert prefill_overhead(2, 512, 16, P) == pytest.approx(0.0552, abs=1e-15)
    assert prefill_overhead(0, 512, 16, P) == 0.0
    assert prefill_overhead(1, 1, 7, P) == pytest.approx(0.002 + 0.00005, abs=1e-15)
    rng = random.Random(0)
    for _ in range(50):                       # Eq. 4 is N-independent in this model
        s, L = rng.randint(0, 9), rng.randint(1, 4096)
        assert prefill_overhead(s, L, rng.randint(0, 500), P) == pytest.approx(prefill_overhead(s, L, 3, P))


def test_expected_reduction_and_net_gain_spec_examples():
    c = SpecCandidate(0, 1, 0.0, p=0.4, t_act=1.5)
    assert expected_reduction([c], 2, 0, 3) == pytest.approx(0.588, abs=1e-12)        # SPEC.md:445 (Eq. 2)
    assert expected_reduction([], 2, 0, 3) == 0.0
    assert expected_reduction([SpecCandidate(0, 1, 0.0, p=1.0, t_act=1.5)], 1, 0, 1) == pytest.approx(1.5)
    with pytest.raises(ValueError):
        expected_reduction([c], 0, 0, 3)
    g = net_gain([c], (16, 2, 0, 0), P, 3)
    assert (g.reduction, g.decode_overhead, g.prefill_overhead) == pytest.approx((0.588, 0.0024, 0.0276))
    assert g.net == pytest.approx(0.558, abs=1e-12)
    assert net_gain([], (16, 2, 0, 0), P, 3).net == 0.0


def test_priority_order_spec_examples():
    a, b = SpecCandidate(1, 1, 5.0), SpecCandidate(2, 4, 1.0)
    assert priority_key(a) < priority_key(b)
    a, b = SpecCandidate(1, 2, 9.0), SpecCandidate(2, 2, 3.0)
    assert priority_key(a) < priority_key(b)
    a, b = SpecCandidate(1, 2, 3.0), SpecCandidate(2, 2, 3.0)
    assert priority_key(a) < priority_key(b)


def test_select_step_spec_examples():
    cfg = SchedulerConfig(k=3, t_w=10.0)
    q = [SpecCandidate(i, 1, float(i)) for i in range(2)]
    r = select_step(q, (16, 2, 0, 0), P, cfg)
    assert len(r.selected) == 2 and q == []
    q = [SpecCandidate(0, 1, 1.0, p=0.0), SpecCandidate(1, 2, 0.0)]
    r = select_step(q, (16, 2, 0, 0), P, cfg)
    assert r.selected == [] and len(q) == 2 and r.returned[0].task_id == 0            # break candidate returned
    q = [SpecCandidate(0, 1, 1.0, wait_time=99.0), SpecCandidate(1, 2, 0.0)]
    r = select_step(q, (16, 2, 0, 0), P, cfg)
    assert [c.task_id for c in r.expired] == [0] and [c.task_id for c in r.selected] == [1]


def _random_queue(rng, n):
    return [SpecCandidate(i, rng.randint(1, 5), rng.uniform(0, 10), wait_time=rng.uniform(0, 2),
                          p=rng.uniform(0, 0.9), t_act=rng.uniform(0.1, 3.0), L_s=rng.randint(16, 1024),
                          l_s=rng.randint(1, 10)) for i in range(n)]


def test_select_step_is_the_greedy_prefix_by_exhaustive_enumeration():
    """S is a prefix of the non-expired priority order, strictly better than
    each strict prefix, and adding the next candidate does not improve it."""
    rng = random.Random(1)
    for trial in range(300):
        n = rng.randint(0, 10)
        q = _random_queue(rng, n)
        cfg = SchedulerConfig(k=rng.randint(1, 4), t_w=1.0)
        params = CostModelParams(base_step_time=0.02, decode_cost_per_request=rng.uniform(0, 3e-3),
                                 decode_knee=rng.randint(1, 64), decode_slowdown=rng.uniform(0, 1),
                                 prefill_fixed_cost=rng.uniform(0, 0.01), prefill_cost_per_token=rng.uniform(0, 1e-4))
        load = (rng.randint(1, 200), rng.randint(1, 20), 0, rng.randint(0, 5))
        order = sorted(q, key=priority_key)
        live = [c for c in order if c.wait_time <= cfg.t_w]
        r = select_step(list(q), load, params, cfg)
        S = r.selected
        assert S == live[:len(S)]
        gains = [net_gain(live[:j], load, params, cfg.k).net for j in range(len(S) + 1)]
        assert all(gains[j + 1] > gains[j] for j in range(len(S)))
        if len(S) < len(live):
            assert net_gain(live[:len(S) + 1], load, params, cfg.k).net <= gains[-1]
        assert all(c.wait_time > cfg.t_w for c in r.expired)
        assert not any(c.wait_time > cfg.t_w for c in S)                                # expiry safety


def test_admitted_count_non_increasing_in_load():
    """identical candidates, N swept across the knee -> |S| non-increasing."""
    params = CostModelParams(decode_cost_per_request=2e-3, decode_knee=64, decode_slowdown=0.5)
    loads = [1, 2, 4, 8, 16, 32, 48, 64, 96, 128, 192, 256]
    got = [s for _, s, _ in admitted_vs_load(params, loads, cand={"t_act": 1.5})]
    # with every main request a candidate, compare the admitted FRACTION of the candidates
    fr = [s / n for s, n in zip(got, loads)]
    assert all(a >= b - 1e-12 for a, b in zip(fr, fr[1:])), fr


def test_forks_that_share_their_prefix_admit_more():
    """Reading F3-a: forks charged gamma_f << gamma (prefix sharing) admit at least as many."""
    shared = CostModelParams(decode_cost_per_request=2e-3, decode_cost_per_fork=1e-4)
    plain = CostModelParams(decode_cost_per_request=2e-3)
    for n in (4, 16, 64, 256):
        a = admitted_vs_load(shared, [n])[0][1]
        b = admitted_vs_load(plain, [n])[0][1]
        assert a >= b


def _synth_table(params, with_forks=False):
    rows = []
    for n in (1, 4, 16, 32, 64, 128, 256):
        rows.append((0, 0, n, hybrid_batch_time((), n, params)))
        for L, c in ((16, 1), (128, 4), (512, 2)):
            rows.append((L, c, n, hybrid_batch_time([(L, c)], n, params)))
        if with_forks:
            for f in (3, 12, 48):
                rows.append((0, 0, n, hybrid_batch_time((), n, params, fork_count=f), f))
    return rows


@pytest.mark.parametrize("with_forks", [False, True])
def test_calibrate_round_trip(with_forks):
    """a table synthesised from known parameters is recovered within 1 %."""
    true = CostModelParams(0.012, 2.3e-4, 64, 0.35, 0.0015, 4e-5, 1.1e-5 if with_forks else None)
    got, rep = calibrate(_synth_table(true, with_forks))
    assert rep["max_rel_err"] < 1e-9
    for f in ("base_step_time", "decode_cost_per_request", "decode_knee", "decode_slowdown", "prefill_fixed_cost",
              "prefill_cost_per_token"):
        assert getattr(got, f) == pytest.approx(getattr(true, f), rel=1e-2), f
    if with_forks:
        assert got.decode_cost_per_fork == pytest.approx(true.decode_cost_per_fork, rel=1e-2)


def test_calibrate_rejects_underdetermined_tables():
    with pytest.raises(CalibrationError):
        calibrate([(0, 0, 16, 0.02)])
    with pytest.raises(CalibrationError):                                              # no hybrid rows
        calibrate([(0, 0, n, 0.02 + n * 1e-4) for n in range(1, 10)])


def test_calibrate_fails_when_the_model_misses_a_row():
    t = _synth_table(P)
    t[3] = (t[3][0], t[3][1], t[3][2], t[3][3] * 3.0)
    with pytest.raises(CalibrationError):
        calibrate(t)
    assert math.isfinite(calibrate(t, max_rel_err=10.0)[1]["max_rel_err"])
