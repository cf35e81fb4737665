"""Batched small-N engine (whole runs on the device, one CTA per run): traces and
bit strings must equal the reference's golden vectors and the per-stage engine
bit for bit; acceptance criterion 2 (100 000 runs of N=15) through it."""
import time

import pytest

from conftest import unhex

pytestmark = pytest.mark.gpu


def E(kind="none", delta=0.0, px=None, py=None, pz=None):
    from paper_2308_05047_b200 import ErrorConfig, ErrorKind, PauliProbs
    return ErrorConfig(ErrorKind[kind], delta, PauliProbs(px, py, pz or 0.0) if px is not None else None)


def engine(N, a, t=None, err=None):
    from paper_2308_05047_b200 import FactoringProblem, IterativeShorEngine, SimulatorOptions
    return IterativeShorEngine(FactoringProblem.make(N, a, t), err or E(),
                               SimulatorOptions(qubit_ceiling=64))


def test_batched_traces_match_reference_golden(cuda_ok, golden):
    groups = {}
    for rec in golden["engine_runs"]:
        groups.setdefault((rec["error"], rec["N"], rec["a"], rec["t"], rec["seed"]), []).append(rec)
    for (ename, N, a, t, seed), recs in groups.items():
        eng = engine(N, a, t, E(**golden["_meta"]["errors"][ename]))
        recs = sorted(recs, key=lambda r: r["idx"])
        runs = eng.run_many(seed, recs[0]["idx"], len(recs))
        for r, rec in zip(runs, recs):
            assert r.bits.j == int(rec["j"]) and r.j_sampled == int(rec["j_sampled"]), (ename, N)
            assert [x.p1 for x in r.trace] == unhex(rec["p1"])
            assert [x.sampled_bit for x in r.trace] == rec["sampled_bit"]
            assert [x.observed_bit for x in r.trace] == rec["observed_bit"]
            assert [int(x.event.classical_flip) for x in r.trace] == rec["classical_flip"]
            assert [int(x.event.quantum_error_branch) for x in r.trace] == rec["quantum_error_branch"]


def test_batched_c2_runs_match_golden(cuda_ok, golden):
    eng = engine(15, 7, 8)
    js = eng.run_batch(2, 0, 64)
    assert js == [int(r["j"]) for r in golden["run_15_c2"]]


@pytest.mark.parametrize("N,a,t,err", [
    (4087, 1001, 20, E()), (4093, 17, 18, E("phase_init", 0.2)), (3599, 7, 16, E("amplitude_init", 0.1)),
    (1001, 10, 20, E("quantum_measure", 0.05, 0.03, 0.02, 0.1)), (35, 4, 11, E("bitflip", 0.1)),
    (21, 2, 9, E("classical_measure", 0.2)), (2047, 3, 20, E()),
])
def test_batched_equals_per_stage_engine(cuda_ok, N, a, t, err):
    eng = engine(N, a, t, err)
    batched = eng.run_many(9, 100, 40)
    seq = eng.run_sequential(9, 100, 40)
    assert [r.bits.j for r in batched] == seq
    for k in (0, 17, 39):
        one = eng.run(9, 100 + k)
        assert [x.p1 for x in batched[k].trace] == [x.p1 for x in one.trace]
        assert batched[k].j_sampled == one.j_sampled


def test_acceptance_c2_statistics_batched(cuda_ok):
    """proj/tests/acceptance/acceptance_main.cpp:93-121 through the batched engine:
    100 000 runs of N=15, a=7, t=8 (seed 2): support {0,64,128,192}, chi-square."""
    eng = engine(15, 7, 8)
    eng.run_batch(2, 0, 1000)  # warm (tables, context)
    t0 = time.perf_counter()
    js = eng.run_batch(2, 0, 100000)
    dt = time.perf_counter() - t0
    counts = {}
    for j in js:
        counts[j] = counts.get(j, 0) + 1
    assert set(counts) <= {0, 64, 128, 192}
    chi2 = sum((counts.get(j, 0) - 25000) ** 2 / 25000 for j in (0, 64, 128, 192))
    assert chi2 < 16.27  # p > 1e-3, 3 dof
    print(f"100000 batched runs of N=15: {dt * 1e3:.1f} ms ({dt / 1e5 * 1e9:.0f} ns/run)")


# ------------------------------------------------------ lockstep (mid-size N)
LOCK_ERRS = [E(), E("classical_measure", 0.05), E("amplitude_init", 0.1), E("phase_init", 0.1),
             E("bitflip", 0.02), E("quantum_measure", 0.02, 0.01, 0.01, 0.0)]


def _trace(r):
    return [(x.p1, x.sampled_bit, x.observed_bit, x.event) for x in r.trace]


@pytest.mark.parametrize("N,a,t", [(4087, 1001, 24), (262139, 4242, 16), (1048351, 12345, 12),
                                   (4194301, 1234567, 10)])
@pytest.mark.parametrize("ei", range(len(LOCK_ERRS)))
def test_lockstep_runs_equal_single_runs(cuda_ok, N, a, t, ei):
    """Shots of a mid-size problem advanced stage by stage together (lockstep.cuh):
    every shot's bit string, sampled bits and p1 trace equal engine.run for it."""
    eng = engine(N, a, t, LOCK_ERRS[ei])
    many = eng.run_many(9, 5, 7)
    for i, r in enumerate(many):
        q = eng.run(9, 5 + i)
        assert r.bits.j == q.bits.j and r.j_sampled == q.j_sampled, i
        assert _trace(r) == _trace(q), i


def test_lockstep_run_problem_matches_reference(cuda_ok, reference):
    """run_problem at L = 12 (N = 4087: t = 24 > the shared-memory batch's 20)
    through the lockstep engine equals the reference's statistics."""
    import paper_2308_05047_b200 as shs
    for i, a in enumerate([1001, 5, 17]):
        prob = shs.FactoringProblem.make(4087, a, p=61, q=67, seed=900 + i)
        got = shs.run_problem(prob, 96)
        ref = reference.run_problem(4087, a, 61, 67, prob.L, prob.t, prob.seed, 96)
        assert (got.success, got.lucky_ne, got.lucky_no, got.lucky_oo, got.fail) == \
            (ref["success"], ref["lucky_ne"], ref["lucky_no"], ref["lucky_oo"], ref["fail"]), a
        assert (got.first_factor_index, got.first_order_index) == \
            (ref["first_factor_index"], ref["first_order_index"])
