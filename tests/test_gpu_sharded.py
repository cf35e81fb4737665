"""The sharded engine's CUDA path (exchange kernels over per-owner pointers,
shard-local probs/collapse, exact digit combine) on ONE GPU with G virtual
shards in one process: every amplitude after every step, p0/p1 and seeded bit
strings must equal the single-GPU engine (SHS_COMBINE_EXACT) bit for bit. No
kernel waits on another shard: each rank's exchange is a separate launch that
only reads the previous stage's completed buffers."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def E(kind="none", delta=0.0, pauli=None):
    from paper_2308_05047_b200 import ErrorConfig, ErrorKind, PauliProbs
    return ErrorConfig(ErrorKind[kind], delta, PauliProbs(*pauli) if pauli else None)


def opts(**kw):
    from paper_2308_05047_b200 import SimulatorOptions
    return SimulatorOptions(**{"qubit_ceiling": 64, "combine": "exact", **kw})


def pair(N, a, t, err, G, tiling="auto"):
    import paper_2308_05047_b200 as shs
    prob = shs.FactoringProblem.make(N, a, t)
    single = shs.IterativeShorEngine(prob, err, opts(tiling=tiling))
    sharded = shs.ShardedShorEngine.virtual(prob, err, opts(tiling=tiling), nshards=G)
    return single, sharded


def full_state(sharded, x, N, stage=False):
    tot = np.zeros(2 * N)
    for sh in sharded.shards:
        arr = sh.stage_read(x, 0, N) if stage else sh.state_read(x, 0, N)
        tot += np.ctypeslib.as_array(arr)
    return tot


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("N,a,t,tiling", [(1048351, 12345, 6, "force"), (4194301, 1234567, 5, "auto"),
                                          (262139, 31337, 6, "off")])
def test_virtual_shards_forced_sequence_bit_exact(cuda_ok, G, N, a, t, tiling):
    err = E("phase_init", 0.1)
    single, sharded = pair(N, a, t, err, G, tiling)
    single.state_init()
    sharded.state_init()
    prefix = 0
    for s in range(t):
        p = single.stage_probs(s, prefix)
        q = sharded.stage_probs(s, prefix)
        assert p == q, (s, p, q)
        for x in (0, 1):
            want = np.ctypeslib.as_array(single.stage_read(x, 0, N))
            assert np.array_equal(full_state(sharded, x, N, stage=True), want)
        b = (s * 7 + 3) % 2
        if p[b] < 1e-300:
            b = 1 - b
        if s + 1 < t:
            single.stage_collapse(b, p[b])
            sharded.stage_collapse(b, q[b])
            for x in (0, 1):
                want = np.ctypeslib.as_array(single.state_read(x, 0, N))
                assert np.array_equal(full_state(sharded, x, N), want)
        prefix |= b << s
    sharded.close()


def same_run(s, r):
    assert s.bits.j == r.bits.j and s.j_sampled == r.j_sampled
    assert [x.p1 for x in s.trace] == [x.p1 for x in r.trace]
    assert [x.sampled_bit for x in s.trace] == [x.sampled_bit for x in r.trace]
    assert [x.observed_bit for x in s.trace] == [x.observed_bit for x in r.trace]
    assert [x.event.classical_flip for x in s.trace] == [x.event.classical_flip for x in r.trace]
    assert [x.event.quantum_error_branch for x in s.trace] == \
        [x.event.quantum_error_branch for x in r.trace]


ERRS = [E(), E("classical_measure", 0.05), E("amplitude_init", 0.1), E("phase_init", 0.2),
        E("bitflip", 0.02), E("quantum_measure", 0.02, (0.01, 0.01, 0.0))]
ERR_IDS = ["none", "classical", "amplitude", "phase", "bitflip", "quantum"]


@pytest.mark.parametrize("err", ERRS, ids=ERR_IDS)
def test_virtual_shards_seeded_runs(cuda_ok, err):
    """Device-resident sharded runs (shs_shards_run: exchange, probs, digit sum and
    the measurement on the device, stages ordered by events) and the host-driven
    per-stage driver equal the single engine."""
    N, a, t = 2097143, 777, 14
    single, sharded = pair(N, a, t, err, 4)
    for idx in range(2):
        r = single.run(11, idx)
        same_run(sharded.run(11, idx), r)
        same_run(sharded.run_stepwise(11, idx), r)
    sharded.close()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_virtual_shards_device_run_shard_counts(cuda_ok, G):
    N, a, t = 4194301, 1234567, 12
    err = E("phase_init", 0.1)
    single, sharded = pair(N, a, t, err, G)
    for idx in range(2):
        same_run(sharded.run(3, idx), single.run(3, idx))
    # the pending state after a device-resident run equals the single engine's
    for x in (0, 1):
        want = np.ctypeslib.as_array(single.stage_read(x, 0, N))
        assert np.array_equal(full_state(sharded, x, N, stage=True), want)
        want = np.ctypeslib.as_array(single.state_read(x, 0, N))
        assert np.array_equal(full_state(sharded, x, N), want)
    sharded.close()


@pytest.mark.parametrize("G", [2, 4])
def test_virtual_shards_kahan_combine_small_n(cuda_ok, G):
    """Below 1025 blocks (AUTO) the shards combine p0/p1 like the reference, with
    the sequential Kahan over all shards' partials: p1 traces equal the single
    engine's (which is bit-identical to the reference there)."""
    import paper_2308_05047_b200 as shs
    for N, a, t in [(262139, 31337, 12), (65521 * 3, 5, 14)]:
        prob = shs.FactoringProblem.make(N, a, t)
        for err in (E(), E("quantum_measure", 0.03, (0.02, 0.01, 0.05))):
            single = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64))
            sharded = shs.ShardedShorEngine.virtual(prob, err, shs.SimulatorOptions(qubit_ceiling=64),
                                                    nshards=G)
            for idx in range(3):
                r = single.run(9, idx)
                same_run(sharded.run(9, idx), r)
                same_run(sharded.run_stepwise(9, idx), r)
            sharded.close()


def test_virtual_shards_config3_run(cuda_ok):
    """Config-3 problem (N = 16777207, t = 48): 8 virtual shards, full run."""
    N, a = 16777207, 2
    single, sharded = pair(N, a, None, E(), 8)
    r = single.run(5, 0)
    same_run(sharded.run(5, 0), r)
    sharded.close()


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0, 0]])
def test_engine_over_devices_equals_single(cuda_ok, devices):
    """Row N1: IterativeShorEngine with SimulatorOptions.devices (shs_options.n_devices)
    is the sharded engine behind the single-engine handle: run(), the step API and
    state reads all equal the one-device engine (virtual shards on this GPU)."""
    import paper_2308_05047_b200 as shs
    N, a, t = 1048351, 12345, 10
    err = E("amplitude_init", 0.1)
    prob = shs.FactoringProblem.make(N, a, t)
    single = shs.IterativeShorEngine(prob, err, opts())
    multi = shs.IterativeShorEngine(prob, err, opts(devices=devices))
    assert multi.devices() == devices and single.devices() == [0]
    for idx in range(3):
        same_run(multi.run(4, idx), single.run(4, idx))
    single.state_init()
    multi.state_init()
    prefix = 0
    rng = np.random.default_rng(1)
    for s in range(t):
        p = single.stage_probs(s, prefix)
        assert multi.stage_probs(s, prefix) == p
        b = int(rng.integers(0, 2)) if min(p) > 1e-6 else int(p[1] > p[0])
        if s + 1 < t:
            single.stage_collapse(b, p[b])
            multi.stage_collapse(b, p[b])
            idx = rng.integers(0, N, 500).astype(np.uint64)
            for x in (0, 1):
                assert np.array_equal(multi.state_gather(x, idx), single.state_gather(x, idx))
                assert np.array_equal(np.ctypeslib.as_array(multi.state_read(x, N - 3000, 3000)),
                                      np.ctypeslib.as_array(single.state_read(x, N - 3000, 3000)))
        prefix |= b << s
    multi.close()


def test_shard_protocol_errors(cuda_ok):
    import paper_2308_05047_b200 as shs
    prob = shs.FactoringProblem.make(1048351, 12345, 6)
    eng = shs.ShardedShorEngine.virtual(prob, E(), opts(), nshards=2)
    eng.state_init()
    eng.stage_probs(0, 0)
    eng.stage_collapse(0, 0.5)
    sh = eng.shards[0]
    assert sh.needs_exchange(1)
    with pytest.raises(ValueError):  # probs before this stage's exchange
        sh.probs(1, 0)
    eng.close()


@pytest.mark.parametrize("G,rounds", [(2, "1"), (3, "2"), (4, "3"), (8, "1"), (5, "4")])
def test_exchange_v2_equals_v1_and_single(cuda_ok, monkeypatch, G, rounds):
    """Device-resident runs with exchange v2 (exchange2.cuh: pack into the
    receivers' streams, unpack through shared-memory transposes, K rounds) equal
    the v1 exchange (SHS_EXCHANGE=1) and the single engine, amplitudes included."""
    import paper_2308_05047_b200 as shs
    monkeypatch.setenv("SHS_X2_ROUNDS", rounds)
    N, a, t = 4194301, 1234567, 10
    err = E("phase_init", 0.1)
    prob = shs.FactoringProblem.make(N, a, t)
    single = shs.IterativeShorEngine(prob, err, opts())
    v2 = shs.ShardedShorEngine.virtual(prob, err, opts(), nshards=G)
    monkeypatch.setenv("SHS_EXCHANGE", "1")
    v1 = shs.ShardedShorEngine.virtual(prob, err, opts(), nshards=G)
    for idx in range(3):
        r = single.run(6, idx)
        same_run(v2.run(6, idx), r)
        same_run(v1.run(6, idx), r)
    for x in (0, 1):  # the pending state after the runs
        want = np.ctypeslib.as_array(single.stage_read(x, 0, N))
        assert np.array_equal(full_state(v2, x, N, stage=True), want)
    v2.close()
    v1.close()


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_sparse_prefix_equals_dense(cuda_ok, G):
    """The sparse prefix of sharded runs (every shard runs the first stages on the
    support, then scatters its range) equals the dense sharded run and the single
    engine (which runs its own sparse prefix) — bits, p1 and the pending state."""
    import paper_2308_05047_b200 as shs
    N, a, t = 4206457, 12345, 26
    for err in (E("phase_init", 0.1), E("quantum_measure", 0.02, (0.01, 0.01, 0.0))):
        prob = shs.FactoringProblem.make(N, a, t)
        single = shs.IterativeShorEngine(prob, err, opts())
        sharded = shs.ShardedShorEngine.virtual(prob, err, opts(), nshards=G)
        assert sharded.sparse_stages() > 0
        for idx in range(2):
            r = single.run(8, idx)
            same_run(sharded.run(8, idx), r)
        for x in (0, 1):
            want = np.ctypeslib.as_array(single.stage_read(x, 0, N))
            assert np.array_equal(full_state(sharded, x, N, stage=True), want)
        sharded.set_sparse(False)
        assert sharded.sparse_stages() == 0
        same_run(sharded.run(8, 5), single.run(8, 5))
        sharded.close()
