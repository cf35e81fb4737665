"""§8 f4: Shor post-processing on the device against the unmodified reference
(oracle/_ref: shor_standard_procedure, proj/src/postprocess.cpp:55-89, and
run_problem, proj/src/harness.cpp:109-148): every outcome field identical
(integer work: bit-exact is the bar)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def fields(o):
    return {"classification": int(o.classification), "r_even": int(o.checks.r_even),
            "a_r_is_one": int(o.checks.a_r_is_one),
            "a_half_not_minus_one": int(o.checks.a_half_not_minus_one),
            "order_match": 2 if o.order_match is None else int(o.order_match),
            "k": o.convergent[0], "r": o.convergent[1], "factors": o.factors}


CASES = [(15, 7, 8, (3, 5)), (21, 2, 9, (3, 7)), (35, 3, 11, (5, 7)), (4087, 1001, 24, (61, 67)),
         (16777207, 2, 48, (4093, 4099)), (4294967213, 5, 64, (57139, 75167)),
         (34359737977, 3, 70, (117517, 292381)), (8589933181, 3974323683, 100, (89597, 95873))]


@pytest.mark.parametrize("N,a,t,pq", CASES)
def test_standard_procedure_matches_reference(cuda_ok, reference, N, a, t, pq):
    import paper_2308_05047_b200 as shs
    from paper_2308_05047_b200.postprocess import outcome_from_record
    rng = random.Random(N ^ t)
    order = shs.multiplicative_order(a, N, pq)
    assert order == reference.multiplicative_order(a, N, *pq)
    js = [0, 1, 2, (1 << t) - 1, 1 << (t - 1)]
    # peaks j ~ k 2^t / r (the interesting continued fractions) and random strings
    js += [(k * (1 << t)) // order + d for k in rng.sample(range(order), min(order, 40))
           for d in (-1, 0, 1)]
    js += [rng.getrandbits(t) for _ in range(200)]
    js = [j for j in js if 0 <= j < (1 << t)]
    arr = np.array([[j & (2**64 - 1), j >> 64] for j in js], dtype=np.uint64)
    for ko in (order, None):
        out = shs.shor_postprocess_array(arr, t, N, a, ko)
        for j, rec in zip(js, out):
            assert fields(outcome_from_record(rec)) == \
                reference.shor_standard_procedure(j, t, N, a, ko), (j, ko)


def test_standard_procedure_errors(cuda_ok):
    import paper_2308_05047_b200 as shs
    with pytest.raises(ValueError):  # convergents: t must be < 128
        shs.shor_standard_procedure(1, 128, 15, 7)
    with pytest.raises(ValueError):  # convergents: j >= 2^t
        shs.shor_standard_procedure(256, 8, 15, 7)
    with pytest.raises(ValueError):
        shs.shor_standard_procedure(1 << 70, 70, 34359737977, 3)
    assert shs.shor_standard_procedure((1 << 70) - 1, 70, 34359737977, 3).convergent[1] >= 1


def _all_bases(N):
    import math
    return [a for a in range(2, N) if math.gcd(a, N) == 1]


@pytest.mark.parametrize("N,pq", [(21, (3, 7)), (35, (5, 7))])
def test_run_problem_matches_reference(cuda_ok, reference, N, pq):
    """Config 2: every coprime base, M shots each, the per-problem statistics
    equal the reference's run_problem (same engine bit strings, same labels)."""
    import paper_2308_05047_b200 as shs
    from oracle import make_error
    M = 256
    for i, a in enumerate(_all_bases(N)):
        prob = shs.FactoringProblem.make(N, a, p=pq[0], q=pq[1], seed=1000 + i)
        got = shs.run_problem(prob, M)
        ref = reference.run_problem(N, a, pq[0], pq[1], prob.L, prob.t, prob.seed, M,
                                    make_error())
        assert got.order == ref["order"] and got.order_solvable == ref["order_solvable"]
        assert (got.success, got.lucky_ne, got.lucky_no, got.lucky_oo, got.fail) == \
            (ref["success"], ref["lucky_ne"], ref["lucky_no"], ref["lucky_oo"], ref["fail"]), a
        assert got.first_factor_index == ref["first_factor_index"]
        assert got.first_order_index == ref["first_order_index"]
        h = got.r_ratio
        assert (h.overflow, h.other, h.total_lucky) == \
            (ref["r_overflow"], ref["r_other"], ref["r_total_lucky"])
        assert h.reciprocal == ref["r_reciprocal"]


def test_run_problem_with_error_model(cuda_ok, reference):
    import paper_2308_05047_b200 as shs
    from oracle import make_error
    prob = shs.FactoringProblem.make(35, 2, p=5, q=7, seed=77)
    err = shs.ErrorConfig(shs.ErrorKind.classical_measure, 0.05)
    got = shs.run_problem(prob, 512, err)
    ref = reference.run_problem(35, 2, 5, 7, prob.L, prob.t, 77, 512,
                                make_error("classical_measure", 0.05))
    assert (got.success, got.lucky_ne, got.lucky_no, got.lucky_oo, got.fail) == \
        (ref["success"], ref["lucky_ne"], ref["lucky_no"], ref["lucky_oo"], ref["fail"])


# ------------------------------------------------------------------ Ekerå
def ekera_fields(o):
    return {"classification": int(o.classification),
            "order_match": 2 if o.order_match is None else int(o.order_match),
            "recovered_order": o.recovered_order, "candidate_offset": o.candidate_offset,
            "k": o.convergent[0], "r": o.convergent[1], "factors": o.factors}


EKERA_CASES = [(15, 7, 8, (3, 5)), (21, 2, 9, (3, 7)), (35, 3, 11, (5, 7)),
               (4087, 1001, 24, (61, 67)), (16777207, 2, 48, (4093, 4099)),
               (4294967213, 5, 64, (57139, 75167))]


@pytest.mark.parametrize("N,a,t,pq", EKERA_CASES)
def test_ekera_matches_reference(cuda_ok, reference, N, a, t, pq):
    """ekera_postprocess (postprocess.cpp:138-171) with the shot's RngStream:
    classification, recovered order, winning offset, convergent, factors and
    order_match identical to the reference for peak, near-peak and random
    bit strings (for_problem parameters: B = L sweeps +-L around j)."""
    import paper_2308_05047_b200 as shs
    from paper_2308_05047_b200.postprocess import ekera_outcome_from_record
    rng = random.Random(7 * N + t)
    L = N.bit_length()
    prm = shs.EkeraParams.for_problem(L, t)
    order = shs.multiplicative_order(a, N, pq)
    js = [0, 1, (1 << t) - 1]
    js += [(k * (1 << t)) // order + d for k in rng.sample(range(order), min(order, 12))
           for d in (0, 3, -L - 1)]
    js += [rng.getrandbits(t) for _ in range(24)]
    js = [j % (1 << t) for j in js]
    arr = np.array([[j & (2**64 - 1), j >> 64] for j in js], dtype=np.uint64)
    seed = 4242
    for ko in (order, None):
        out = shs.ekera_postprocess_array(arr, t, N, a, prm, seed, 100, ko)
        for i, (j, rec) in enumerate(zip(js, out)):
            ref = reference.ekera_postprocess(j, t, N, a, (prm.B, prm.c, prm.k, prm.varsigma,
                                                            prm.m, prm.ell), seed, 100 + i, ko)
            assert ekera_fields(ekera_outcome_from_record(rec)) == ref, (j, ko)


@pytest.mark.parametrize("N,pq", [(21, (3, 7)), (35, (5, 7))])
def test_run_problem_ekera_matches_reference(cuda_ok, reference, N, pq):
    import paper_2308_05047_b200 as shs
    for i, a in enumerate(_all_bases(N)[:8]):
        prob = shs.FactoringProblem.make(N, a, p=pq[0], q=pq[1], seed=500 + i)
        got = shs.run_problem(prob, 256, post_mode="ekera")
        ref = reference.run_problem(N, a, pq[0], pq[1], prob.L, prob.t, prob.seed, 256,
                                    post_mode="ekera")
        assert (got.success, got.fail, got.first_factor_index, got.first_order_index) == \
            (ref["success"], ref["fail"], ref["first_factor_index"], ref["first_order_index"]), a


def test_factorize_and_rho_budget_match_reference(cuda_ok, reference):
    """factorize (numtheory.cpp:170-187) on the device equals the reference's, and
    its Pollard-rho budget runs out exactly where the reference's does
    (FactorizationTimeoutError, numtheory.cpp:137, 149): for each composite the
    smallest budget the reference needs is found by bisection; the device
    succeeds with it and times out with one step less."""
    import random

    import paper_2308_05047_b200 as shs
    from oracle import OracleError
    rng = random.Random(4)

    def prime(bits):
        while True:
            c = rng.getrandbits(bits) | (1 << (bits - 1)) | 1
            if all(c % d for d in range(3, 2000, 2)) and pow(2, c - 1, c) == 1:
                return c

    cases = [prime(20) * prime(21), prime(28) * prime(29), prime(31) * prime(32),
             prime(12) * prime(13) * prime(14), 2 ** 5 * 97 * prime(25) * prime(26),
             prime(16) ** 2 * prime(20), 1, 97, 2 ** 63 + 1]
    for n in cases:
        want = reference.factorize(n)
        assert shs.factorize(n) == want, n
        lo, hi = 0, 10_000_000  # the reference: hi works, lo - 1 ... find the least budget
        try:
            reference.factorize(n, 0)
            need = 0
        except OracleError as e:
            assert e.code == 9
            while hi - lo > 1:
                mid = (lo + hi) // 2
                try:
                    reference.factorize(n, mid)
                    hi = mid
                except OracleError:
                    lo = mid
            need = hi
        assert shs.factorize(n, max(need, 0) or 1) == want if need else True
        if need > 1:
            assert shs.factorize(n, need) == want
            with pytest.raises(shs.FactorizationTimeoutError):
                shs.factorize(n, need - 1)


def test_ekera_rho_budget_timeout(cuda_ok):
    """recover_order's factorize() budget in the device Ekerå pipeline: a tiny
    budget makes ekera_postprocess raise FactorizationTimeoutError as the
    reference's would (postprocess.cpp:113 -> numtheory.cpp:137)."""
    import numpy as np

    import paper_2308_05047_b200 as shs
    N, a, t = 1048351, 12345, 40
    L = N.bit_length()
    params = shs.EkeraParams.for_problem(L, t)
    j = np.array([[123456789, 0]], dtype=np.uint64)
    shs.ekera_postprocess_array(j, t, N, a, params, 1, 0)  # default budget: fine
    import dataclasses
    tight = dataclasses.replace(params, rho_budget=1)
    hit = False
    for x in range(1, 400):  # some convergent denominator is composite with a large factor
        j = np.array([[x * 7919 % (1 << t), 0]], dtype=np.uint64)
        try:
            shs.ekera_postprocess_array(j, t, N, a, tight, 1, 0)
        except shs.FactorizationTimeoutError:
            hit = True
            break
    assert hit
