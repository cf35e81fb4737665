"""Device-resident runs (engine.cu engine_run_device, the default run path):
measurement, collapse group and next-stage scalars decided on the device
(measure.cuh, k_finalize_measure), the host one stage behind supplying the two
candidate phases. Checked against the host-driven loop (SHS_HOST_MEASURE=1,
the step-by-step twin of proj/src/statevector.cpp:323-412) and the C oracle:
identical bit strings, sampled bits, p1 traces, and the same pending final
stage afterwards."""
import numpy as np
import pytest

from test_gpu_parity import E, engine, oracle_err

pytestmark = pytest.mark.gpu

ERRS = [E(), E("classical_measure", 0.05), E("amplitude_init", 0.1), E("phase_init", 0.1),
        E("bitflip", 0.02), E("quantum_measure", 0.02, 0.01, 0.01, 0.0)]


def pair(monkeypatch, N, a, t, err, **opt):
    dev = engine(N, a, t, err, **opt)
    monkeypatch.setenv("SHS_HOST_MEASURE", "1")
    host = engine(N, a, t, err, **opt)
    monkeypatch.delenv("SHS_HOST_MEASURE")
    return dev, host


def same_run(r, q):
    assert r.bits.j == q.bits.j and r.j_sampled == q.j_sampled
    assert [(x.p1, x.sampled_bit, x.observed_bit, x.event) for x in r.trace] == \
           [(x.p1, x.sampled_bit, x.observed_bit, x.event) for x in q.trace]


@pytest.mark.parametrize("N,a,t", [(15, 7, 8), (4087, 1001, 24), (262139, 4242, 12),
                                   (4194301, 1234567, 10)])
@pytest.mark.parametrize("ei", range(len(ERRS)))
def test_device_run_equals_host_run(cuda_ok, monkeypatch, N, a, t, ei):
    err = ERRS[ei]
    dev, host = pair(monkeypatch, N, a, t, err)
    for idx in range(3):
        same_run(dev.run(11, idx), host.run(11, idx))
    # the engine is left with stage t-1 pending, as after the host loop
    n = min(N, 4096)
    for x in (0, 1):
        assert np.array_equal(np.asarray(dev.stage_read(x, 0, n)),
                              np.asarray(host.stage_read(x, 0, n)))


@pytest.mark.parametrize("ei", range(len(ERRS)))
def test_device_run_vs_oracle_tiled(cuda_ok, oracle, ei):
    """Tiled stages (N = 2^22) with every error model: bit strings equal the
    oracle's (exact combine on both sides)."""
    err = ERRS[ei]
    N, a, t = 4194301, 1234567, 8
    eng = engine(N, a, t, err)
    assert sum(eng.tile_plan(s)["tiled"] for s in range(1, t)) >= 1
    orc = oracle.engine(N, a, N.bit_length(), t, oracle_err(err))
    for idx in range(2):
        r = eng.run(3, idx)
        o = orc.run(3, idx, 1)
        assert r.bits.j == o["j"] and r.j_sampled == o["j_sampled"]
        assert [tr.p1 for tr in r.trace] == o["p1"]


def test_device_run_interleaves_with_step_api(cuda_ok, monkeypatch):
    """run() then the step API then run() again: no state leaks between them."""
    dev, host = pair(monkeypatch, 262139, 4242, 12, E("phase_init", 0.1))
    a = dev.run(5, 0)
    dev.state_init()
    p = dev.stage_probs(0, 0)
    dev.stage_collapse(1, p[1])
    b = dev.run(5, 1)
    same_run(a, host.run(5, 0))
    same_run(b, host.run(5, 1))


# ---------------------------------------------------------------- sparse prefix
def _runs(eng, seed, n):
    return [eng.run(seed, i) for i in range(n)]


@pytest.mark.parametrize("N,a,t", [(16777207, 2, None), (16777207, 3, None), (16777207, 2, 10),
                                   (67108859, 5, 20)])
@pytest.mark.parametrize("ei", [0, 3, 5])
def test_sparse_prefix_equals_dense(cuda_ok, monkeypatch, N, a, t, ei):
    """The first stages on the support of the state (sparse.cuh) against the
    dense device-resident run and the host-driven loop: identical bit strings,
    sampled bits and p1 traces (every stage, every error model)."""
    err = ERRS[ei]
    sp, host = pair(monkeypatch, N, a, t, err)
    dense = engine(N, a, t, err)
    dense.set_sparse(False)
    assert sp.sparse_stages() >= 8 and dense.sparse_stages() == 0
    for r, d, h in zip(_runs(sp, 19, 2), _runs(dense, 19, 2), _runs(host, 19, 2)):
        same_run(r, d)
        same_run(r, h)
    # the pending last stage is the same dense state
    for first in (0, N // 2, N - 4096):
        for x in (0, 1):
            assert np.array_equal(np.asarray(sp.stage_read(x, first, 4096)),
                                  np.asarray(dense.stage_read(x, first, 4096)))


def test_sparse_prefix_stops_before_the_orbit_wraps(cuda_ok):
    """a of small order (1364 | ord): the host's baby-step giant-step check caps
    the sparse prefix where 2^(s+1) would exceed ord(A_s); results still equal
    the dense run."""
    import paper_2308_05047_b200 as shs
    N, lam = 16777207, 2794836
    a = pow(2, lam // 1364, N)
    o = shs.multiplicative_order(a, N, (4093, 4099))
    assert o <= 1364
    sp = engine(N, a)
    dense = engine(N, a)
    dense.set_sparse(False)
    n = sp.sparse_stages()
    pows = sp.stage_multipliers()
    for s in range(n):  # no wrap inside the prefix
        assert shs.multiplicative_order(pows[s], N, (4093, 4099)) >= 2 ** (s + 1)
    for r, d in zip(_runs(sp, 3, 3), _runs(dense, 3, 3)):
        same_run(r, d)
