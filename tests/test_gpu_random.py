"""Randomized parity sweep: fresh (N, a, t, error model, seed, index) draws,
every kernel path (per-stage direct gather, forced sorted-residue tiles,
batched whole-run kernel, virtual shards) against the C oracle — bit strings,
sampled strings and p1 traces identical (Kahan combine where the reference's
applies, exact combine for the sharded path)."""
import math
import random

import pytest

pytestmark = pytest.mark.gpu

ERRS = [("none", 0.0, None), ("classical_measure", 0.1, None), ("amplitude_init", 0.2, None),
        ("phase_init", 0.15, None), ("bitflip", 0.05, None),
        ("quantum_measure", 0.04, (0.03, 0.01, 0.02))]


def draw(rng, lo, hi):
    while True:
        N = rng.randrange(lo, hi) | 1
        a = rng.randrange(2, N - 1)
        if math.gcd(a, N) == 1:
            return N, a


@pytest.mark.parametrize("seed", range(6))
def test_random_problems_all_paths(cuda_ok, oracle, seed):
    import paper_2308_05047_b200 as shs
    from oracle import make_error
    rng = random.Random(1000 + seed)
    for trial in range(4):
        N, a = draw(rng, 300000, 1 << 21) if trial % 2 else draw(rng, 1000, 4000)
        t = rng.randrange(6, 13)
        kind, delta, pauli = ERRS[(seed + trial) % len(ERRS)]
        err = shs.ErrorConfig(shs.ErrorKind[kind], delta, shs.PauliProbs(*pauli) if pauli else None)
        oe = make_error(kind, delta, *(pauli or (0.0, 0.0, 0.0)))
        prob = shs.FactoringProblem.make(N, a, t)
        orc = oracle.engine(N, a, N.bit_length(), t, oe)
        s0, idx = rng.getrandbits(64), rng.randrange(1 << 32)
        want = orc.run(s0, idx, 0 if N <= 262144 else 1)
        wantx = orc.run(s0, idx, 1)
        paths = []
        for tiling in ("off", "force"):
            eng = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64, tiling=tiling))
            paths.append((f"per-stage/{tiling}", eng.run(s0, idx), want))
            if N <= 4096:
                paths.append(("batched", eng.run_many(s0, idx, 1)[0], want))
        if N > 4096:
            sh = shs.ShardedShorEngine.virtual(prob, err, shs.SimulatorOptions(
                qubit_ceiling=64, combine="exact", tiling="force"), nshards=rng.choice([2, 3, 4]))
            paths.append(("sharded", sh.run(s0, idx), wantx))
            sh.close()
        for name, r, w in paths:
            ctx = (name, N, a, t, kind, s0, idx)
            assert r.bits.j == w["j"] and r.j_sampled == w["j_sampled"], ctx
            assert [x.p1 for x in r.trace] == w["p1"], ctx
