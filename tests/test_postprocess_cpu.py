"""§8 f4 host side on the CPU: the ground-truth order and the note_outcome
tally (proj/src/harness.cpp:82-104) against the unmodified reference. The
outcomes fed to the tally are the reference's own shor_standard_procedure
results for the reference engine's shots, so the tally alone is under test
(the device post-processing is tests/test_gpu_postprocess.py)."""
import numpy as np
import pytest


@pytest.mark.parametrize("a,N,pq", [(7, 15, (3, 5)), (2, 21, (3, 7)), (3, 35, (5, 7)),
                                    (2, 16777207, (4093, 4099)), (5, 4294967213, (57139, 75167)),
                                    (3, 34359737977, (117517, 292381))])
def test_multiplicative_order(reference, a, N, pq):
    from paper_2308_05047_b200.postprocess import multiplicative_order
    assert multiplicative_order(a, N, pq) == reference.multiplicative_order(a, N, *pq)
    if N < (1 << 20):
        assert multiplicative_order(a, N) == reference.multiplicative_order(a, N)


@pytest.mark.parametrize("N,a,pq,seed", [(21, 2, (3, 7), 5), (35, 3, (5, 7), 9), (35, 4, (5, 7), 1)])
def test_tally_matches_run_problem(reference, N, a, pq, seed):
    from paper_2308_05047_b200 import FactoringProblem
    from paper_2308_05047_b200.postprocess import OUTCOME_DTYPE, ProblemResult, tally
    from paper_2308_05047_b200.postprocess import multiplicative_order
    M = 200
    prob = FactoringProblem.make(N, a, p=pq[0], q=pq[1], seed=seed)
    order = multiplicative_order(a, N, pq)
    eng = reference.engine(N, a, prob.L, prob.t)
    out = np.zeros(M, dtype=OUTCOME_DTYPE)
    for m in range(M):
        o = reference.shor_standard_procedure(eng.run(seed, m)["j"], prob.t, N, a, order)
        out[m]["classification"] = o["classification"]
        out[m]["r"] = (o["r"], 0)
        out[m]["n_factors"] = len(o["factors"])
    res = tally(ProblemResult(problem=prob, M=M, order=order), out)
    ref = reference.run_problem(N, a, pq[0], pq[1], prob.L, prob.t, seed, M)
    assert (res.success, res.lucky_ne, res.lucky_no, res.lucky_oo, res.fail) == \
        (ref["success"], ref["lucky_ne"], ref["lucky_no"], ref["lucky_oo"], ref["fail"])
    assert res.first_factor_index == ref["first_factor_index"]
    assert res.first_order_index == ref["first_order_index"]
    assert (res.r_ratio.overflow, res.r_ratio.other, res.r_ratio.total_lucky) == \
        (ref["r_overflow"], ref["r_other"], ref["r_total_lucky"])
    assert res.r_ratio.reciprocal == ref["r_reciprocal"]
