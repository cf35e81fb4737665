"""Parity at the benchmark configurations (BASELINE.json configs 3 and 4, and the
u64 index range just above 2^32 that config 5 depends on).

* Config 3 (N = 16777207 = 4093 * 4099, t = 48): full seeded runs through
  ``IterativeShorEngine.run`` (AUTO combine, sparse prefix on, as a user runs
  it) against the live UNMODIFIED reference (oracle/_ref, workers = nproc) for
  the paper's six error models, two bases, two bit-string indices each: bit
  strings, sampled strings, per-stage bits and error flags identical; every p1
  within 1 ulp of the reference's sequential Kahan combine
  (proj/src/statevector.cpp:32-40) and ``==`` the oracle's exact combine (the
  engine's AUTO mode above 1024 blocks).
* Config 4 (N = 4294967213, t = 64, 2 x 68.7 GB): the dense round-robin tiled
  kernels (k_tiled<., false>; and the opt-in orbit-compressed stages,
  k_tiled<true, false, true>) under a seeded forced sequence, stages 0..22,
  against the sparse-support oracle (oracle/shor_oracle.c so_sparse_*, itself
  pinned to the dense oracle in tests/test_oracle_pinned.py): p0/p1 ``==`` per
  stage (they sum every one of the 16.7 M block partials), every support
  amplitude ``==`` after every collapse, random off-support windows exactly 0.
* N = 4296381013 = 63719 * 67427 > 2^32 (L = 33, 2 x 68.7 GB): the same check
  for stages 0..20, so the u64 index paths run with real data.
"""
import gc
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def E(kind="none", delta=0.0, px=None, py=None, pz=None):
    from paper_2308_05047_b200 import ErrorConfig, ErrorKind, PauliProbs
    pauli = PauliProbs(px, py, pz or 0.0) if px is not None else None
    return ErrorConfig(ErrorKind[kind], delta, pauli)


def oracle_err(err):
    from oracle import make_error
    p = err.pauli
    return make_error(err.kind.name, err.delta, p.px if p else 0.0, p.py if p else 0.0,
                      p.pz if p else 0.0)


# the paper's error models: init errors at delta = 0.1, measurement
# and bit-flip errors at p = 0.01 with the quantum channel's px = py = delta / 2
# (acceptance_main.cpp:367-378)
ERRORS = {
    "none": E(),
    "amplitude_init": E("amplitude_init", 0.1),
    "phase_init": E("phase_init", 0.1),
    "classical_measure": E("classical_measure", 0.01),
    "quantum_measure": E("quantum_measure", 0.01, 0.005, 0.005, 0.0),
    "bitflip": E("bitflip", 0.01),
}


def ulps(a, b):
    if a == b:
        return 0
    return abs(a - b) / math.ulp(max(abs(a), abs(b)))


def _engine(N, a, t, err):
    from paper_2308_05047_b200 import FactoringProblem, IterativeShorEngine, SimulatorOptions
    return IterativeShorEngine(FactoringProblem.make(N, a, t), err,
                               SimulatorOptions(qubit_ceiling=64))


@pytest.mark.slow
@pytest.mark.parametrize("a", [2, 1234567])
def test_c3_full_runs_vs_live_reference(cuda_ok, oracle, reference, a):
    N, t = 16777207, 48
    L = N.bit_length()
    workers = os.cpu_count() or 1
    for name, err in ERRORS.items():
        oe = oracle_err(err)
        eng = _engine(N, a, t, err)
        assert eng.sparse_stages() > 0  # the default run path, sparse prefix included
        ref = reference.engine(N, a, L, t, oe, shard_count=4, workers=workers, qubit_ceiling=33)
        orc = oracle.engine(N, a, L, t, oe)
        for idx in (0, 1):
            seed = 1000 + idx
            r = eng.run(seed, idx)
            o = ref.run(seed, idx)
            assert r.bits.j == o["j"], (name, a, idx)
            assert r.j_sampled == o["j_sampled"], (name, a, idx)
            assert [x.sampled_bit for x in r.trace] == o["sampled_bit"], (name, a, idx)
            assert [x.observed_bit for x in r.trace] == o["observed_bit"], (name, a, idx)
            assert [int(x.event.classical_flip) for x in r.trace] == o["classical_flip"]
            assert [int(x.event.quantum_error_branch) for x in r.trace] == \
                o["quantum_error_branch"]
            p1 = [x.p1 for x in r.trace]
            worst = max(ulps(x, y) for x, y in zip(p1, o["p1"]))
            assert worst <= 1, (name, a, idx, worst)
            ex = orc.run(seed, idx, 1)  # exact combine of the same block partials
            assert p1 == ex["p1"] and ex["j"] == r.bits.j, (name, a, idx)
        del ref, orc
        eng.close()
        gc.collect()


def _forced_dense_vs_sparse_oracle(oracle, N, a, t, stages, err_name, seed=7, idx=3, orbit=False):
    """Dense step API (tiled kernels; orbit=True: the orbit-compressed stages) vs the
    sparse-support oracle on a seeded forced sequence (the reference's own sampling
    decides every bit)."""
    err = ERRORS[err_name]
    oe = oracle_err(err)
    eng = _engine(N, a, t, err)
    eng.set_sparse(False)
    eng.set_orbit(orbit)
    if orbit:
        assert eng.orbit_info()["stages"] > 0
    so = oracle.sparse(N, a, N.bit_length(), t, oe)
    rng = np.random.default_rng(N % 1000003)
    eng.state_init()
    so.state_init()
    prefix = 0
    kept = []
    try:
        for s in range(stages):
            p0, p1 = eng.stage_probs(s, prefix)
            q0, q1 = so.stage_probs(s, prefix, 1)  # exact combine (16.7 M blocks)
            assert (p0, p1) == (q0, q1), (N, s, p0, p1, q0, q1)
            mr = oracle.sample(q1, seed, idx, s, oe)  # sampled, observed, branch, flip
            src = 1 - mr[0] if mr[2] else mr[0]
            eng.stage_collapse(src, p1 if src else p0)
            so.collapse(src, q1 if src else q0)
            kept.append(src)
            for x in (0, 1):
                z, v = so.state(x)
                got = eng.state_gather(x, z)
                assert np.array_equal(got, v), (N, s, x, int(np.sum(got != v)))
            zs = z.astype(np.int64)
            for first in [0, N - 4096] + [int(f) for f in rng.integers(0, N - 4096, 4)]:
                w = np.frombuffer(eng.state_read(1, first, 4096), dtype=np.float64)
                w = w.reshape(-1, 2).copy()
                inside = zs[(zs >= first) & (zs < first + 4096)] - first
                w[inside] = 0.0
                assert not np.any(w), (N, s, first)
            prefix |= mr[1] << s
    finally:
        eng.close()
        del so
        gc.collect()
    return kept


@pytest.mark.slow
@pytest.mark.parametrize("orbit", [False, True])
def test_c4_dense_stages_vs_sparse_support_oracle(cuda_ok, oracle, orbit):
    N, a, t = 4294967213, 5, 64
    eng = _engine(N, a, t, ERRORS["none"])
    plans = [eng.tile_plan(s) for s in range(1, 23)]
    eng.close()
    assert all(p["tiled"] for p in plans)  # the round-robin tiled kernels are what runs
    kept = _forced_dense_vs_sparse_oracle(oracle, N, a, t, 23, "phase_init", orbit=orbit)
    assert 0 < sum(kept) < len(kept)  # both collapse paths (speculative h0 and h1) ran


@pytest.mark.slow
def test_above_2_32_dense_stages_vs_sparse_support_oracle(cuda_ok, oracle):
    N, a = 4296381013, 5  # 63719 * 67427, L = 33
    assert N > 1 << 32
    t = 66
    kept = _forced_dense_vs_sparse_oracle(oracle, N, a, t, 21, "amplitude_init")
    assert 0 < sum(kept) < len(kept)


@pytest.mark.slow
def test_c4_sharded_run_equals_single(cuda_ok):
    """Config 4 through the multi-device engine (row N1): the state split over 2
    virtual shards of this GPU (2 x 2 x 34.4 GB + exchange-v2 receive slots, K
    rounds sized to the remaining memory), a full device-resident run with the
    sharded sparse prefix and exchange v2 — bits, sampled bits and every p1 equal
    the single engine's run (exact combine at 16.7 M blocks in both)."""
    import paper_2308_05047_b200 as shs
    N, a = 4294967213, 5
    err = ERRORS["quantum_measure"]
    prob = shs.FactoringProblem.make(N, a)
    single = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64))
    r = single.run(31, 7)
    single.close()
    gc.collect()
    multi = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64,
                                                                  devices=[0, 0]))
    assert multi.devices() == [0, 0] and multi.sparse_stages() > 0
    s = multi.run(31, 7)
    multi.close()
    gc.collect()
    assert s.bits.j == r.bits.j and s.j_sampled == r.j_sampled
    assert [x.p1 for x in s.trace] == [x.p1 for x in r.trace]
    assert [x.event.quantum_error_branch for x in s.trace] == \
        [x.event.quantum_error_branch for x in r.trace]
