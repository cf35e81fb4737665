"""Orbit-compressed stages (paper_2308_05047_b200/csrc/orbit.cuh).

The work register's support never leaves the orbit <a> (statevector.cpp:326-345:
start |1>, gathers through powers of a), so the engine stores and sweeps only its
r = ord_N(a) members on stages with whole-band tile plans. These tests check that
the compressed engine is indistinguishable from the dense one:
* full device-resident runs (sparse prefix -> compressed scatter, compressed
  stages, expansion to dense for the last small-multiplier stages): identical bit
  strings, sampled bits, error branches and every p1 (==);
* the host-driven step API (dense -> compressed transition after stage 0):
  p0 / p1 ==, and the state windows and post-Hadamard windows == at every stage;
* the orbit index: r = the multiplicative order of a.
Config 4 itself goes through the compressed path in test_gpu_bench_parity.py
(the dense tiled stages against the sparse-support oracle, every support
amplitude after every collapse).
"""
import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N30, A30, R30 = 1073217479, 2, 536575980  # 32749 * 32771, ord(2) from bench.py's n30


def _engine(N, a, err=None):
    import paper_2308_05047_b200 as shs
    prob = shs.FactoringProblem.make(N, a)
    eng = shs.IterativeShorEngine(prob, err or shs.ErrorConfig(),
                                  shs.SimulatorOptions(qubit_ceiling=64))
    eng.set_orbit(True)
    return eng


def test_orbit_info_n30(cuda_ok):
    eng = _engine(N30, A30)
    info = eng.orbit_info()
    assert info["r"] == R30
    assert info["stages"] >= 20 and info["first"] >= 1
    eng.set_orbit(False)
    assert eng.orbit_info()["r"] == 0
    eng.close()


def test_orbit_runs_equal_dense_n30(cuda_ok):
    import paper_2308_05047_b200 as shs
    err = shs.ErrorConfig(shs.ErrorKind.quantum_measure, 0.01, shs.PauliProbs(0.005, 0.005, 0.0))
    eng = _engine(N30, A30, err)
    assert eng.orbit_info()["stages"] > 0 and eng.sparse_stages() > 0
    runs = [(7, i) for i in range(3)]
    orb = [eng.run(s, i) for s, i in runs]
    eng.set_sparse(False)  # dense stage 0 .. : dense -> compressed transition in run()
    orb_nosparse = eng.run(7, 0)
    eng.set_sparse(True)
    eng.set_orbit(False)
    dense = [eng.run(s, i) for s, i in runs]
    eng.close()
    gc.collect()
    for o, d in zip(orb, dense):
        assert o.bits.j == d.bits.j and o.j_sampled == d.j_sampled
        assert [x.p1 for x in o.trace] == [x.p1 for x in d.trace]
        assert [x.event.quantum_error_branch for x in o.trace] == \
            [x.event.quantum_error_branch for x in d.trace]
    assert orb_nosparse.bits.j == dense[0].bits.j
    assert [x.p1 for x in orb_nosparse.trace] == [x.p1 for x in dense[0].trace]


def test_orbit_step_api_states_equal_dense_n30(cuda_ok, oracle):
    """Forced sequence through the step API on two engines (compressed / dense):
    p0, p1 and windows of the state and of the post-Hadamard groups, every stage."""
    from paper_2308_05047_b200 import ErrorConfig
    from oracle import make_error
    a_eng = _engine(N30, A30)
    b_eng = _engine(N30, A30)
    b_eng.set_orbit(False)
    oe = make_error("none", 0.0, 0.0, 0.0, 0.0)
    t = a_eng.problem.t
    rng = np.random.default_rng(5)
    firsts = [0, N30 - 2048] + [int(f) for f in rng.integers(0, N30 - 2048, 3)]
    try:
        a_eng.state_init()
        b_eng.state_init()
        prefix = 0
        for s in range(t):
            pa = a_eng.stage_probs(s, prefix)
            pb = b_eng.stage_probs(s, prefix)
            assert pa == pb, (s, pa, pb)
            for f in firsts[:2]:
                for x in (0, 1):
                    wa = np.frombuffer(a_eng.stage_read(x, f, 2048), dtype=np.float64)
                    wb = np.frombuffer(b_eng.stage_read(x, f, 2048), dtype=np.float64)
                    assert np.array_equal(wa, wb), (s, f, x)
            if s + 1 == t:
                break
            mr = oracle.sample(pa[1], 11, 3, s, oe)
            src = 1 - mr[0] if mr[2] else mr[0]
            a_eng.stage_collapse(src, pa[1] if src else pa[0])
            b_eng.stage_collapse(src, pb[1] if src else pb[0])
            for f in firsts:
                for x in (0, 1):
                    wa = np.frombuffer(a_eng.state_read(x, f, 2048), dtype=np.float64)
                    wb = np.frombuffer(b_eng.state_read(x, f, 2048), dtype=np.float64)
                    assert np.array_equal(wa, wb), (s, f, x)
            idx = np.sort(rng.integers(0, N30, 4096).astype(np.uint64))
            assert np.array_equal(a_eng.state_gather(1, idx), b_eng.state_gather(1, idx)), s
            prefix |= mr[1] << s
    finally:
        a_eng.close()
        b_eng.close()
        gc.collect()


@pytest.mark.parametrize("N,a,r", [
    (1087482493, 2, 181236090),  # 32971 * 32983: the orbit is N / 6
    (1074262927, 2, 523488),     # 32719 * 32833: N / 2052 (slots pack 4 near-empty sub-chunks)
])
def test_orbit_low_density_runs_equal_dense(cuda_ok, N, a, r):
    """Orbits much smaller than N / 2: the compressed stages pack up to four
    sub-chunks per slot; runs with and without the sparse prefix equal the
    dense engine's."""
    import paper_2308_05047_b200 as shs
    err = shs.ErrorConfig(shs.ErrorKind.phase_init, 0.1)
    eng = _engine(N, a, err)
    assert eng.orbit_info()["r"] == r and eng.orbit_info()["stages"] > 0
    got = []
    for sparse in (True, False):
        eng.set_sparse(sparse)
        got.append(eng.run(5, 1))
    eng.set_orbit(False)
    want = []
    for sparse in (True, False):
        eng.set_sparse(sparse)
        want.append(eng.run(5, 1))
    eng.close()
    gc.collect()
    for g, w in zip(got, want):
        assert g.bits.j == w.bits.j and g.j_sampled == w.j_sampled
        assert [x.p1 for x in g.trace] == [x.p1 for x in w.trace]


@pytest.mark.parametrize("N,a", [
    (4186067, 2),      # 2039 * 2053, just below 2^22: compressed from 2^21 (orbit.cuh kOrbitMinN)
    (16777207, 1234567),  # config 3's size (bench.py config3_error_models)
])
def test_orbit_default_on_mid_sizes_equal_dense(cuda_ok, N, a):
    """The compressed stages are the default from 2^21 (where AUTO tiling gives the
    stages tile plans); runs under every error kind equal the dense engine's."""
    import paper_2308_05047_b200 as shs
    kinds = [shs.ErrorConfig(),
             shs.ErrorConfig(shs.ErrorKind.quantum_measure, 0.01, shs.PauliProbs(0.005, 0.005, 0.0)),
             shs.ErrorConfig(shs.ErrorKind.amplitude_init, 0.01),
             shs.ErrorConfig(shs.ErrorKind.bitflip, 0.01)]
    for err in kinds:
        prob = shs.FactoringProblem.make(N, a)
        eng = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64))
        assert eng.orbit_info()["stages"] > 0  # on by default
        got = [eng.run(3, i) for i in range(3)]
        eng.set_orbit(False)
        want = [eng.run(3, i) for i in range(3)]
        eng.close()
        for g, w in zip(got, want):
            assert g.bits.j == w.bits.j and g.j_sampled == w.j_sampled
            assert [x.p1 for x in g.trace] == [x.p1 for x in w.trace]
    gc.collect()
