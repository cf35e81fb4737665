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


@pytest.mark.parametrize("err", [E(), E("classical_measure", 0.05), E("amplitude_init", 0.1),
                                 E("bitflip", 0.02), E("quantum_measure", 0.02, (0.01, 0.01, 0.0))],
                         ids=["none", "classical", "amplitude", "bitflip", "quantum"])
def test_virtual_shards_seeded_runs(cuda_ok, err):
    N, a, t = 2097143, 777, 14
    single, sharded = pair(N, a, t, err, 4)
    for idx in range(2):
        r = single.run(11, idx)
        s = sharded.run(11, idx)
        assert s.bits.j == r.bits.j and s.j_sampled == r.j_sampled
        assert [x.p1 for x in s.trace] == [x.p1 for x in r.trace]
        assert [x.observed_bit for x in s.trace] == [x.observed_bit for x in r.trace]
    sharded.close()


def test_virtual_shards_config3_run(cuda_ok):
    """Config-3 problem (N = 16777207, t = 48): 8 virtual shards, full run."""
    N, a = 16777207, 2
    single, sharded = pair(N, a, None, E(), 8)
    r = single.run(5, 0)
    s = sharded.run(5, 0)
    assert s.bits.j == r.bits.j and [x.p1 for x in s.trace] == [x.p1 for x in r.trace]
    sharded.close()


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
