"""The C oracle (oracle/shor_oracle.c) pinned to the reference: its golden
vectors (tests/golden, produced by the unmodified reference) and, where
oracle/_ref is built, the live reference library on fresh seeded inputs.
CPU only."""
import math
import random
from fractions import Fraction

import pytest

from conftest import unhex

def oerr(golden, name):
    from oracle import make_error
    return make_error(**golden["_meta"]["errors"][name])


def test_philox_kat(oracle, golden):
    # proj/tests/test_util.cpp:82-89
    assert oracle.philox(0, [0, 0, 0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    for v in golden["philox"]["vectors"]:
        assert oracle.philox(v["key"], v["ctr"]) == v["out"]


def test_fig3_plan(oracle, golden):
    pf = golden["plan_fig3"]
    assert oracle.index_map(16, 55, 0, 55) == pf["gather"]
    assert pf["gather"][48] == 3
    assert sum(map(sum, pf["pair_counts"])) == 55
    assert all(row[7] == 0 for row in pf["pair_counts"])
    inv = oracle.mod_inverse(16, 55)
    back = oracle.index_map(inv, 55, 0, 55)
    assert [back[g] for g in pf["gather"]] == list(range(55))
    for p in golden["plans"]:
        g = oracle.index_map(p["a_pow"], p["N"], 0, p["N"])
        assert g[:64] == p["head"] and g[-64:] == p["tail"]
        assert sum((i + 1) * x for i, x in enumerate(g)) % (2**61 - 1) == p["checksum"]


def _cmp(run, rec):
    assert run["j"] == int(rec["j"]) and run["j_sampled"] == int(rec["j_sampled"])
    assert run["p1"] == unhex(rec["p1"])
    for k in ("sampled_bit", "observed_bit", "classical_flip", "quantum_error_branch"):
        assert run[k] == rec[k], k


def test_engine_runs_golden(oracle, golden):
    cache = {}
    for rec in golden["engine_runs"]:
        key = (rec["error"], rec["N"], rec["a"])
        if key not in cache:
            cache[key] = oracle.engine(rec["N"], rec["a"], rec["N"].bit_length(), rec["t"],
                                       oerr(golden, rec["error"]))
        _cmp(cache[key].run(rec["seed"], rec["idx"]), rec)


@pytest.mark.parametrize("case,N,a,t", [("run_4087", 4087, 1001, 24), ("run_8051", 8051, 2024, 26),
                                        ("run_15_c2", 15, 7, 8)])
def test_byte_stable_golden(oracle, golden, case, N, a, t):
    eng = oracle.engine(N, a, N.bit_length(), t)
    for rec in golden[case]:
        _cmp(eng.run(rec["seed"], rec["idx"]), rec)


def test_multipliers(oracle, golden):
    assert oracle.engine(15, 7, 4, 8).multipliers() == golden["multipliers_15_7"]


def test_forced_sequences_golden(oracle, golden):
    for fs in golden["forced"]:
        eng = oracle.engine(fs["N"], fs["a"], fs["N"].bit_length(), fs["t"], oerr(golden, fs["error"]))
        eng.state_init()
        prefix = 0
        for st in fs["steps"]:
            p0, p1 = eng.stage_probs(st["s"], prefix, 0)
            assert p0 == float.fromhex(st["p0"]) and p1 == float.fromhex(st["p1"])
            for x, key in ((0, "g0"), (1, "g1")):
                assert list(eng.stage_read(x, 0, 64)) == unhex(st["post_h"][key])
            if "post_reset" in st:
                b = st["bit"]
                eng.collapse(b, p1 if b else p0)
                for x, key in ((0, "g0"), (1, "g1")):
                    assert list(eng.state_read(x, 0, 64)) == unhex(st["post_reset"][key])
            prefix |= st["bit"] << st["s"]


def test_exhaustive_peaks_and_sampling(oracle, golden):
    """N=15, a=7, t=8 distribution sits on multiples of 64 (test_statevector.cpp:357-364);
    oracle samples follow it (criterion-2 style chi-square)."""
    dist = unhex(golden["exhaustive_15_7_8"])
    for j, p in enumerate(dist):
        assert abs(p - (0.25 if j % 64 == 0 else 0.0)) < 1e-12
    eng = oracle.engine(15, 7, 4, 8)
    counts = {}
    n = 4000
    for i in range(n):
        j = eng.run(2, i)["j"]
        counts[j] = counts.get(j, 0) + 1
    assert set(counts) <= {0, 64, 128, 192}
    chi2 = sum((counts.get(j, 0) - n / 4) ** 2 / (n / 4) for j in (0, 64, 128, 192))
    assert chi2 < 16.27  # p > 1e-3 at 3 dof


def test_exact_sum_is_correctly_rounded(oracle):
    rng = random.Random(5)
    for trial in range(200):
        k = rng.randrange(1, 300)
        scale = 2.0 ** rng.randrange(-60, 3)
        vals = [rng.random() * scale * (2.0 ** rng.randrange(-40, 1)) for _ in range(k)]
        if trial % 7 == 0:
            vals += [5e-324, 2.2250738585072014e-308, 0.0]
        exact = sum(Fraction(v) for v in vals)
        assert oracle.exact_sum(vals) == float(exact)  # float(Fraction) rounds to nearest-even
    assert oracle.exact_sum([]) == 0.0
    assert oracle.exact_sum([1.0, 2.0 ** -53]) == 1.0  # tie -> even
    assert oracle.exact_sum([1.0, 2.0 ** -53, 2.0 ** -200]) == 1.0 + 2.0 ** -52


def test_sampling_matches_reference_live(oracle, reference):
    from oracle import make_error
    errs = [make_error(), make_error("classical_measure", 0.3), make_error("bitflip", 0.1),
            make_error("quantum_measure", 0.1, 0.05, 0.05, 0.1),
            make_error("quantum_measure", 0.5, 0.25, 0.25, 0.0)]
    rng = random.Random(3)
    for err in errs:
        for _ in range(300):
            p1 = rng.choice([0.0, 1.0, 0.5, rng.random()])
            seed, idx, st = rng.getrandbits(64), rng.getrandbits(32), rng.randrange(128)
            r = reference.sample(p1, seed, idx, st, err)
            o = oracle.sample(p1, seed, idx, st, err)
            assert (o[0], o[1], o[2], o[3]) == (r[0], r[1], r[2], r[3])


def test_random_problems_match_reference_live(oracle, reference):
    """Fresh (N, a, error, seed) draws, oracle vs the unmodified reference engine."""
    from oracle import make_error
    rng = random.Random(2308)
    errs = [make_error(), make_error("classical_measure", 0.1), make_error("amplitude_init", 0.2),
            make_error("phase_init", 0.05), make_error("bitflip", 0.05),
            make_error("quantum_measure", 0.04, 0.03, 0.01, 0.02)]
    done = 0
    while done < 24:
        N = rng.randrange(15, 20000) | 1
        a = rng.randrange(2, N - 1)
        if math.gcd(a, N) != 1:
            continue
        t = rng.randrange(4, 16)
        err = errs[done % len(errs)]
        L = N.bit_length()
        o = oracle.engine(N, a, L, t, err)
        r = reference.engine(N, a, L, t, err, qubit_ceiling=33)
        assert o.multipliers() == r.multipliers()
        for idx in range(3):
            seed = rng.getrandbits(64)
            try:
                want = r.run(seed, idx)
            except Exception as exc:  # degenerate branches must fail identically
                with pytest.raises(Exception):
                    o.run(seed, idx)
                continue
            assert o.run(seed, idx) == want
        done += 1


def test_index_map_matches_reference_live(oracle, reference):
    rng = random.Random(11)
    for _ in range(20):
        N = rng.randrange(3, 1 << 16)
        a = rng.randrange(1, N)
        if math.gcd(a, N) != 1:
            continue
        n = N.bit_length() + 1
        plan = reference.plan(a, N, n, 2)
        assert oracle.index_map(a, N, 0, N) == plan["gather"]


def _sparse_vs_dense(oracle, reference, N, a, t, err, seed, bits_rng):
    """so_sparse (the config-4 checker) == so_engine (and the reference's per-gate
    state) on a seeded forced sequence: p0/p1 in both combine modes, every support
    amplitude, and zero off the support."""
    import numpy as np
    L = N.bit_length()
    d = oracle.engine(N, a, L, t, err)
    sp = oracle.sparse(N, a, L, t, err)
    d.state_init()
    sp.state_init()
    prefix = 0
    for s in range(t):
        for mode in (1, 0):  # exact first: the Kahan call leaves the pending state the same
            q = d.stage_probs(s, prefix, mode)
            r = sp.stage_probs(s, prefix, mode)
            assert q == r, (N, s, mode)
        b = bits_rng.randrange(2) if min(q) > 1e-6 else int(q[1] > q[0])
        d.collapse(b, q[b])
        sp.collapse(b, r[b])
        for x in (0, 1):
            z, v = sp.state(x)
            full = np.frombuffer(d.state_read(x, 0, N), dtype=np.float64).reshape(-1, 2)
            assert np.array_equal(full[z.astype(np.int64)].ravel(), v), (N, s, x)
            mask = np.ones(N, bool)
            mask[z.astype(np.int64)] = False
            assert not np.any(full[mask]), (N, s, x)
        prefix |= b << s


def test_sparse_support_oracle_equals_dense(oracle, reference):
    from oracle import make_error
    rng = random.Random(5)
    cases = [(1048351, 12345, 14, make_error("phase_init", 0.1)),      # threaded dense path
             (196597, 3, 16, make_error()),                            # orbit wraps early
             (4087, 1001, 24, make_error("amplitude_init", 0.15)),     # support saturates
             (15, 7, 8, make_error())]                                 # identity stages
    for N, a, t, err in cases:
        _sparse_vs_dense(oracle, reference, N, a, t, err, 3, rng)
