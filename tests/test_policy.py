"""Prefetch/eviction policy parity: tests/test_prefetch.cpp re-expressed, plus
bit-exact doubles and picks against the compiled reference."""
import json
import math
import os
import random

import pytest

from paper_2512_20210_b200 import (AdapterDynamics, PrefetchPolicy, Residency, ValidationError,
                                   eviction_score, plan_evictions, recency_score,
                                   scored_residents, select_prefetch)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def resident_at(last, decayed, p):  # test_prefetch.cpp:12-20
    return AdapterDynamics(status=Residency.resident, last_access_ms=last, decayed_count=decayed,
                           decay_stamp_ms=0.0 if last < 0 else last, prediction=p)


def test_policy_validation():  # :24-32
    p = PrefetchPolicy()
    p.validate()
    p.theta = 1.0
    with pytest.raises(ValidationError):
        p.validate()
    p = PrefetchPolicy(alpha=0.0, beta=0.0, gamma=0.0)
    with pytest.raises(ValidationError):
        p.validate()


def test_score_arithmetic_example():  # :34-45
    policy = PrefetchPolicy(alpha=1.0, beta=1.0, gamma=1.0)
    now = 100_000.0
    d = resident_at(now - policy.tau_ms * math.log(2.0), 0.0, 0.9)
    d.decayed_count = 0.2
    d.decay_stamp_ms = now
    assert eviction_score(d, policy, now, 1.0) == pytest.approx(1.6, rel=1e-9)


def test_alpha_only_is_lru():  # :47-62
    policy = PrefetchPolicy(alpha=1.0, beta=0.0, gamma=0.0)
    dyn = [resident_at(t, 5.0, 0.9) for t in (10_000.0, 400_000.0, 250_000.0, 499_000.0)]
    assert [k for _, k in scored_residents(dyn, policy, 500_000.0)] == [0, 2, 1, 3]


def test_monotone():  # :64-83
    policy = PrefetchPolicy()
    now = 1_000_000.0
    base = resident_at(now - 30_000, 4.0, 0.5)
    s0 = eviction_score(base, policy, now, 10.0)
    for field, val in (("last_access_ms", now - 10_000), ("decayed_count", 8.0),
                       ("prediction", 0.9)):
        d = resident_at(now - 30_000, 4.0, 0.5)
        setattr(d, field, val)
        assert eviction_score(d, policy, now, 10.0) > s0


def test_select_prefetch_golden():  # :110-142 via tests/golden/policy_golden.json
    with open(os.path.join(GOLDEN, "policy_golden.json")) as f:
        g = json.load(f)
    pol = PrefetchPolicy(theta=0.8)
    dyn = [AdapterDynamics() for _ in range(4)]
    units = [2, 2, 2, 2]
    assert select_prefetch([0.8, 0.8000001, 0.1, 0.0], dyn, pol, units, 100) == \
        g["strict_threshold"] == [1]
    assert select_prefetch([0.9, 0.7, 0.95, -1.0], dyn, pol, units, 2) == g["cap2"] == [2]
    assert select_prefetch([0.9, 0.7, 0.95, -1.0], dyn, pol, units, 4) == g["cap4"] == [2, 0]
    dyn[2].status = Residency.staging
    dyn[0].transfer_active = True
    assert select_prefetch([0.9, 0.85, 0.95, 0.99], dyn, pol, units, 100) == \
        g["staging_excluded"] == [3, 1]
    dyn = [resident_at(1.0, 1.0, 0.5) for _ in range(4)]
    assert select_prefetch([0.9, 0.95, 0.99, 0.85], dyn, pol, units, 100) == []


def test_plan_evictions_golden():  # :167-189
    with open(os.path.join(GOLDEN, "policy_golden.json")) as f:
        g = json.load(f)
    b = [100, 50, 200, 80]
    p = plan_evictions(120, 0, [1, 3, 0, 2], b)
    assert (p.victims, p.satisfied) == tuple(g["evict_120"]) == ([1, 3], True)
    p = plan_evictions(40, 50, [0, 1, 2, 3], b)
    assert (p.victims, p.satisfied) == tuple(g["evict_noop"]) == ([], True)
    p = plan_evictions(1000, 0, [0, 1], b)
    assert (p.victims, p.satisfied) == tuple(g["evict_unsat"]) == ([], False)


def test_random_cases_bit_exact_golden():
    """50 random states: scores/orderings/picks equal the reference's doubles."""
    with open(os.path.join(GOLDEN, "policy_golden.json")) as f:
        g = json.load(f)
    for case in g["random"]:
        dyn = [AdapterDynamics(status=Residency(d["status"]), last_access_ms=d["last_access_ms"],
                               decayed_count=d["decayed_count"],
                               decay_stamp_ms=d["decay_stamp_ms"], prediction=d["prediction"],
                               busy=d["busy"], transfer_active=d["transfer_active"])
               for d in case["dyn"]]
        pol = PrefetchPolicy(**case["policy"])
        assert [list(x) for x in scored_residents(dyn, pol, case["now"])] == \
            [list(x) for x in case["scored"]]
        assert select_prefetch(case["probs"], dyn, pol, case["units"], case["budget"]) == \
            case["picks"]
        assert [eviction_score(d, pol, case["now"], 5.0) for d in dyn] == case["scores"]


def test_random_parity_live_reference(ref):
    rng = random.Random(77)
    for _ in range(300):
        n = 1 + rng.randrange(16)
        dyn = [AdapterDynamics(status=Residency(rng.randrange(3)),
                               last_access_ms=rng.random() * 3e5 - 1e4,
                               decayed_count=rng.random() * 20, decay_stamp_ms=rng.random() * 2e5,
                               prediction=rng.random(), transfer_active=rng.random() < 0.3)
               for _ in range(n)]
        pol = PrefetchPolicy(theta=0.05 + 0.9 * rng.random(), alpha=rng.random(),
                             beta=rng.random(), gamma=rng.random() + 1e-3,
                             tau_ms=1 + rng.random() * 1e5,
                             freq_half_life_ms=1 + rng.random() * 1e5)
        now = 2e5 + rng.random() * 1e5
        probs = [rng.random() for _ in range(n + rng.randrange(3) - 1)]
        units = [rng.randrange(1, 9) for _ in range(n)]
        budget = rng.randrange(30)
        assert select_prefetch(probs, dyn, pol, units, budget) == \
            ref.select_prefetch(probs, dyn, pol, units, budget)
        assert scored_residents(dyn, pol, now) == ref.scored_residents(dyn, pol, now)
        for d in dyn:
            assert eviction_score(d, pol, now, 3.0) == ref.eviction_score(d, pol, now, 3.0)
            assert d.decayed_at(now, pol.freq_half_life_ms) == ref.decayed_at(
                d, now, pol.freq_half_life_ms)
        elig = [k for _, k in scored_residents(dyn, pol, now)]
        bf = [rng.randrange(1, 100) for _ in range(n)]
        need, free = rng.randrange(200), rng.randrange(50)
        p = plan_evictions(need, free, elig, bf)
        assert (p.victims, p.satisfied) == ref.plan_evictions(need, free, elig, bf)


def test_recency_and_decay():  # :191-205
    assert recency_score(-1.0, 100.0, 60_000.0) == 0.0
    assert recency_score(100.0, 100.0, 60_000.0) == 1.0
    assert recency_score(0.0, 60_000.0, 60_000.0) == pytest.approx(math.exp(-1.0))
    d = AdapterDynamics()
    d.record_access(0.0, 120_000.0)
    d.record_access(0.0, 120_000.0)
    assert d.decayed_at(0.0, 120_000.0) == pytest.approx(2.0)
    assert d.decayed_at(120_000.0, 120_000.0) == pytest.approx(1.0)
    assert d.decayed_at(240_000.0, 120_000.0) == pytest.approx(0.5)
