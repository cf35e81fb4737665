"""exhaustive_joint_distribution on the device vs the reference (golden vectors
and, where oracle/_ref is present, the live reference library): bit-identical
distributions, the reference's limits and node-budget errors."""
import math
import os
import random

import pytest

from conftest import unhex

pytestmark = pytest.mark.gpu


def E(kind="none", delta=0.0, px=None, py=None, pz=None):
    from paper_2308_05047_b200 import ErrorConfig, ErrorKind, PauliProbs
    return ErrorConfig(ErrorKind[kind], delta,
                       PauliProbs(px, py, pz or 0.0) if px is not None else None)


def dist(N, a, t, err=None, **kw):
    import paper_2308_05047_b200 as shs
    return shs.exhaustive_joint_distribution(shs.FactoringProblem.make(N, a, t), err or E(), **kw)


def test_exhaustive_matches_golden(cuda_ok, golden):
    assert dist(15, 7, 8) == unhex(golden["exhaustive_15_7_8"])
    for case in golden["exhaustive_cases"]:
        got = dist(case["N"], case["a"], case["t"], E(**case["error"]))
        assert got == unhex(case["dist"]), case["name"]


def test_exhaustive_matches_live_reference(cuda_ok, reference):
    from oracle import make_error
    rng = random.Random(77)
    kinds = [dict(kind="none"), dict(kind="classical_measure", delta=0.15),
             dict(kind="quantum_measure", delta=0.06, px=0.04, py=0.02, pz=0.05),
             dict(kind="bitflip", delta=0.03), dict(kind="amplitude_init", delta=0.25),
             dict(kind="phase_init", delta=0.4)]
    done = 0
    while done < 18:
        N = rng.randrange(15, 2048) | 1
        a = rng.randrange(2, N - 1)
        if math.gcd(a, N) != 1:
            continue
        ekw = kinds[done % len(kinds)]
        t = rng.randrange(4, 9) if ekw["kind"] in ("classical_measure", "quantum_measure") else \
            rng.randrange(5, 13)
        want = reference.exhaustive(N, a, N.bit_length(), t, make_error(**ekw))
        got = dist(N, a, t, E(**ekw))
        assert got == want, (N, a, t, ekw)
        done += 1


def test_exhaustive_limits_and_budget(cuda_ok):
    from paper_2308_05047_b200 import BudgetExceededError, ConfigError
    with pytest.raises(BudgetExceededError):  # t <= 14 (statevector.cpp:536-537)
        dist(15, 7, 16)
    with pytest.raises(BudgetExceededError):  # n <= 12
        dist(4093, 3, 10)
    # node budget: N=15, a=7, t=8 costs 9 path nodes + 4 leaves = 13 ticks (six identity
    # stages have p1 = 0), so 13 suffices and 12 throws, as in the reference's recurse()
    assert abs(sum(dist(15, 7, 8, node_budget=13)) - 1.0) < 1e-12
    with pytest.raises(BudgetExceededError):
        dist(15, 7, 8, node_budget=12)
    with pytest.raises(ConfigError):
        dist(15, 7, 8, E("bitflip", 2.0))
    d = dist(1021, 5, 14)  # the reference's largest: t = 14
    assert abs(sum(d) - 1.0) < 1e-10
