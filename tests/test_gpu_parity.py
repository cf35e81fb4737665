"""GPU parity: the CUDA engine (through the C ABI) against the reference's own
golden vectors (tests/golden, generated from the unmodified reference) and the
C oracle (oracle/shor_oracle.c) on identical seeded inputs.

Gates (BASELINE.json north_star):
  * index map bit-exact;
  * amplitudes after every step bit-identical (<= 1e-12 relative L2 is the
    stated tolerance) under the reference's forced measurement sequences;
  * bit strings identical for seeded runs; p1 traces bit-identical where the
    reference's sequential Kahan combine is used (AUTO at small N) and within
    1 ulp where the exact combine is used.
"""
import math
import random

import numpy as np
import pytest

from conftest import unhex

pytestmark = pytest.mark.gpu

REL_L2_TOL = 1e-12  # north_star amplitude tolerance


def E(kind="none", delta=0.0, px=None, py=None, pz=None):
    from paper_2308_05047_b200 import ErrorConfig, ErrorKind, PauliProbs
    pauli = PauliProbs(px, py, pz or 0.0) if px is not None else None
    return ErrorConfig(ErrorKind[kind], delta, pauli)


def golden_error(g, name):
    kw = dict(g["_meta"]["errors"][name])
    return E(**kw)


def engine(N, a, t=None, err=None, **opt):
    from paper_2308_05047_b200 import FactoringProblem, IterativeShorEngine, SimulatorOptions
    o = SimulatorOptions(**{"qubit_ceiling": 64, **opt})
    return IterativeShorEngine(FactoringProblem.make(N, a, t), err or E(), o)


def oracle_err(err):
    from oracle import make_error
    p = err.pauli
    return make_error(err.kind.name, err.delta, p.px if p else 0.0, p.py if p else 0.0,
                      p.pz if p else 0.0)


def ulps(a, b):
    if a == b:
        return 0
    return abs(a - b) / math.ulp(max(abs(a), abs(b)))


def arr(x):
    return np.ctypeslib.as_array(x) if not isinstance(x, (list, np.ndarray)) else np.asarray(x)


def rel_l2(x, y):
    x, y = arr(x), arr(y)
    den = float(np.sum(y * y))
    num = float(np.sum((x - y) ** 2))
    return math.sqrt(num / den) if den else math.sqrt(num)


# ---------------------------------------------------------------- index map
@pytest.mark.parametrize("N,a_pow", [(55, 16), (15, 4), (4087, 1001), (1048351, 12345),
                                     (16777207, 9876543), (4294967213, 3000000019),
                                     (34359737977, 12345678901)])
def test_index_map_bit_exact(cuda_ok, N, a_pow):
    from oracle import Oracle
    o = Oracle()
    a_inv = o.mod_inverse(a_pow, N)
    eng = engine(N, a_pow, t=1)
    rng = random.Random(N)
    windows = [(0, min(N, 5000)), (max(0, N - 3000), min(N, 3000))]
    for _ in range(4):
        first = rng.randrange(0, max(1, N - 4096))
        windows.append((first, min(4096, N - first)))
    for first, count in windows:
        got = list(eng.index_map(0, first, count))
        want = [(a_inv * z) % N for z in range(first, first + count)]
        assert got == want, (N, a_pow, first)


def test_index_map_matches_reference_plan(cuda_ok, golden):
    pf = golden["plan_fig3"]
    eng = engine(pf["N"], pf["a_pow"], t=1)
    assert list(eng.index_map(0, 0, pf["N"])) == pf["gather"]
    for p in golden["plans"]:
        eng = engine(p["N"], p["a_pow"], t=1)
        N = p["N"]
        g = list(eng.index_map(0, 0, N))
        if p["a_pow"] % N == 1:
            assert g == list(range(N))
        assert g[:64] == p["head"] and g[-64:] == p["tail"]
        assert sum((i + 1) * x for i, x in enumerate(g)) % (2**61 - 1) == p["checksum"]


# ---------------------------------------------------------- seeded runs
def _check_run(res, rec):
    assert res.bits.j == int(rec["j"])
    assert res.j_sampled == int(rec["j_sampled"])
    assert [tr.p1 for tr in res.trace] == unhex(rec["p1"])  # bit-identical
    assert [tr.sampled_bit for tr in res.trace] == rec["sampled_bit"]
    assert [tr.observed_bit for tr in res.trace] == rec["observed_bit"]
    assert [int(tr.event.classical_flip) for tr in res.trace] == rec["classical_flip"]
    assert [int(tr.event.quantum_error_branch) for tr in res.trace] == rec["quantum_error_branch"]


def test_engine_runs_match_reference_golden(cuda_ok, golden):
    """proj/tests/test_statevector.cpp:236-279 pin set, against the reference's outputs."""
    cache = {}
    for rec in golden["engine_runs"]:
        key = (rec["error"], rec["N"], rec["a"])
        if key not in cache:
            cache[key] = engine(rec["N"], rec["a"], rec["t"], golden_error(golden, rec["error"]))
        _check_run(cache[key].run(rec["seed"], rec["idx"]), rec)


@pytest.mark.parametrize("case,N,a,t", [("run_4087", 4087, 1001, 24), ("run_8051", 8051, 2024, 26),
                                        ("run_15_c2", 15, 7, 8)])
def test_byte_stable_runs(cuda_ok, golden, case, N, a, t):
    for shards in (2, 16):
        eng = engine(N, a, t, shard_count=shards)
        for rec in golden[case]:
            _check_run(eng.run(rec["seed"], rec["idx"]), rec)


def test_multipliers_and_identity_stages(cuda_ok, golden):
    eng = engine(15, 7, 8)
    assert eng.stage_multipliers() == golden["multipliers_15_7"]
    # stage-0 p1 in {0, 1/2}, proj/tests/test_statevector.cpp:188-208
    for N, a in [(15, 7), (21, 2), (55, 16), (493, 5)]:
        e = engine(N, a)
        r = e.run(99, 0)
        want = 0.0 if e.stage_multipliers()[0] == 1 else 0.5
        assert abs(r.trace[0].p1 - want) <= 1e-12


# ------------------------------------------------------ forced sequences
def test_forced_sequences_amplitudes_bit_exact(cuda_ok, golden):
    """CS3 per-gate path (oracle, phase, Hadamard, measure, reset_top) driven
    through the step API; amplitudes after every step vs the reference."""
    for fs in golden["forced"]:
        eng = engine(fs["N"], fs["a"], fs["t"], golden_error(golden, fs["error"]))
        eng.state_init()
        prefix = 0
        for st in fs["steps"]:
            p0, p1 = eng.stage_probs(st["s"], prefix)
            assert p0 == float.fromhex(st["p0"]) and p1 == float.fromhex(st["p1"])
            for x, key in ((0, "g0"), (1, "g1")):
                got = list(eng.stage_read(x, 0, 64))
                want = unhex(st["post_h"][key])
                assert got == want, (fs["error"], st["s"], key)
            if "post_reset" in st:
                b = st["bit"]
                eng.stage_collapse(b, p1 if b else p0)
                for x, key in ((0, "g0"), (1, "g1")):
                    got = list(eng.state_read(x, 0, 64))
                    assert got == unhex(st["post_reset"][key]), (fs["error"], st["s"], key)
            prefix |= st["bit"] << st["s"]


@pytest.mark.parametrize("tiling", ["off", "force"])
@pytest.mark.parametrize("N,a,t,err", [
    (1048351, 12345, 6, E()),
    (1048351, 777, 5, E("phase_init", 0.1)),
    (262139, 31337, 6, E("amplitude_init", 0.1)),
    (4194301, 5, 4, E("quantum_measure", 0.01, 0.005, 0.005, 0.0)),
    (4194301, 1234567, 5, E("classical_measure", 0.05)),
])
def test_forced_sequence_vs_oracle_full_state(cuda_ok, oracle, N, a, t, err, tiling):
    """Whole-state comparison (every amplitude) after every step at sizes the
    oracle finishes in seconds; random forced branches; direct-gather and
    sorted-residue-tile kernels."""
    eng = engine(N, a, t, err, combine="kahan", tiling=tiling)
    tiled = [eng.tile_plan(s)["tiled"] for s in range(t)]
    assert not tiled[0]
    if tiling == "off":
        assert not any(tiled)
    orc = oracle.engine(N, a, N.bit_length(), t, oracle_err(err))
    eng.state_init()
    orc.state_init()
    prefix = 0
    rng = random.Random(N + t)
    for s in range(t):
        p0, p1 = eng.stage_probs(s, prefix)
        q0, q1 = orc.stage_probs(s, prefix, 0)
        assert (p0, p1) == (q0, q1)
        d0, d1 = eng.block_sums()
        o0, o1 = orc.block_sums()
        assert list(d0) == list(o0) and list(d1) == list(o1)  # reference block partials, bit-identical
        for x in (0, 1):
            got = arr(eng.stage_read(x, 0, N))
            want = arr(orc.stage_read(x, 0, N))
            assert rel_l2(got, want) <= REL_L2_TOL
            assert np.array_equal(got, want)
        b = rng.randrange(2)
        if (p1 if b else p0) < 1e-300:
            b = 1 - b
        if s + 1 < t:
            eng.stage_collapse(b, p1 if b else p0)
            orc.collapse(b, p1 if b else p0)
            for x in (0, 1):
                got = arr(eng.state_read(x, 0, N))
                want = arr(orc.state_read(x, 0, N))
                assert np.array_equal(got, want)
        prefix |= b << s


def test_exact_combine_is_correctly_rounded(cuda_ok, oracle):
    N, a = 16777207, 1234567
    eng = engine(N, a, 5, combine="exact")
    orc = oracle.engine(N, a, N.bit_length(), 5)
    eng.state_init()
    orc.state_init()
    prefix = 0
    for s in range(5):
        p0, p1 = eng.stage_probs(s, prefix)
        q0, q1 = orc.stage_probs(s, prefix, 1)  # oracle exact sum of the same partials
        k0, k1 = orc.stage_probs(s, prefix, 0)  # reference Kahan
        assert (p0, p1) == (q0, q1)
        assert ulps(p0, k0) <= 1 and ulps(p1, k1) <= 1
        b = s & 1
        eng.stage_collapse(b, p1 if b else p0)
        orc.collapse(b, p1 if b else p0)
        prefix |= b << s


def test_seeded_runs_vs_oracle_mid_size(cuda_ok, oracle):
    """Full seeded runs at N ~ 2^16..2^18 with every error model: identical bit strings."""
    errs = [E(), E("classical_measure", 0.05), E("amplitude_init", 0.1), E("phase_init", 0.1),
            E("bitflip", 0.02), E("quantum_measure", 0.02, 0.01, 0.01, 0.0)]
    for err in errs:
        for N, a in [(65521 * 3, 101), (262139, 4242)]:
            t = 12
            eng = engine(N, a, t, err)
            orc = oracle.engine(N, a, N.bit_length(), t, oracle_err(err))
            for idx in range(2):
                r = eng.run(5, idx)
                o = orc.run(5, idx, 0)
                assert r.bits.j == o["j"] and r.j_sampled == o["j_sampled"]
                assert [tr.p1 for tr in r.trace] == o["p1"]


# ------------------------------------------------------- error behaviour
def test_errors_are_raised(cuda_ok):
    from paper_2308_05047_b200 import (CeilingExceededError, ConfigError, DegenerateBranchError,
                                       FactoringProblem, IterativeShorEngine, NotInvertibleError,
                                       SimulatorOptions)
    with pytest.raises(NotInvertibleError) as ei:
        IterativeShorEngine(FactoringProblem.make(15, 6, 8), E(), SimulatorOptions())
    assert ei.value.gcd == 3
    with pytest.raises(CeilingExceededError):
        IterativeShorEngine(FactoringProblem.make(4087, 1001, 24), E(),
                            SimulatorOptions(qubit_ceiling=12))
    with pytest.raises(ConfigError):
        IterativeShorEngine(FactoringProblem.make(15, 7), E("bitflip", 1.5), SimulatorOptions())
    with pytest.raises(ValueError):
        IterativeShorEngine(FactoringProblem.make(15, 7), E(), SimulatorOptions(shard_count=3))
    eng = engine(15, 7, 8)
    eng.state_init()
    eng.stage_probs(0, 0)
    with pytest.raises(DegenerateBranchError):  # proj/tests/test_statevector.cpp:219
        eng.stage_collapse(1, 0.0)


@pytest.mark.parametrize("N,a,split", [(16777207, 1234567, ""), (268435247, 3, ""),
                                       (268435247, 3, "0"), (16777207, 1234567, "0")])
def test_tiled_work_split_vs_direct(cuda_ok, monkeypatch, N, a, split):
    """The tiled kernels in both work-split variants against the direct-gather
    kernels: bit-identical 256-block partials and states. Default: few bands
    (CTA ranges cut inside bands); SHS_TILE_SPLIT=0 forces whole bands handed
    out dynamically (the config-4 variant; at N = 2^28, 1024 bands for 148 CTAs)."""
    if split:
        monkeypatch.setenv("SHS_TILE_SPLIT", split)
    rng = np.random.default_rng(N)
    tiled = engine(N, a)
    monkeypatch.delenv("SHS_TILE_SPLIT", raising=False)
    direct = engine(N, a, tiling="off")
    t = 6  # the first stages of the full schedule: "random" multipliers
    assert sum(tiled.tile_plan(s)["tiled"] for s in range(1, t)) >= t - 2
    tiled.state_init()
    direct.state_init()
    prefix = 0
    for s in range(t):
        p = tiled.stage_probs(s, prefix)
        assert p == direct.stage_probs(s, prefix), s
        d0, d1 = tiled.block_sums()
        e0, e1 = direct.block_sums()
        assert np.array_equal(d0, e0) and np.array_equal(d1, e1), s
        b = int(rng.integers(2)) if min(p) > 1e-300 else int(p[1] > p[0])
        if s + 1 == t:
            break
        tiled.stage_collapse(b, p[b])
        direct.stage_collapse(b, p[b])
        for first in [0, N - 4096] + [int(x) for x in rng.integers(0, N - 4096, 6)]:
            for x in (0, 1):
                assert np.array_equal(arr(tiled.state_read(x, first, 4096)),
                                      arr(direct.state_read(x, first, 4096))), (s, first)
        prefix |= b << s


@pytest.mark.parametrize("N,a,split,tiling", [(16777207, 1234567, "", "auto"),
                                              (268435247, 3, "0", "auto"),
                                              (1048351, 12345, "", "off"),
                                              (16777207, 5, "", "off")])
def test_speculative_group0_write(cuda_ok, monkeypatch, N, a, split, tiling):
    """Tiled probs passes also store h0 into the successor buffer, so a stage
    that keeps group 0 skips its collapse: identical block sums, states and
    seeded runs to the engine with every collapse launched (SHS_SPEC=0), for
    both work-split variants, forced branches of both kinds and device-resident
    runs (where the collapse kernel returns at once on group 0); tiled and
    direct kernels (gather; a = 5: the staged-stream small multipliers)."""
    if split:
        monkeypatch.setenv("SHS_TILE_SPLIT", split)
    opt = {} if tiling == "auto" else {"tiling": tiling}
    spec = engine(N, a, 8, **opt)
    monkeypatch.setenv("SHS_SPEC", "0")
    full = engine(N, a, 8, **opt)
    monkeypatch.delenv("SHS_SPEC", raising=False)
    monkeypatch.delenv("SHS_TILE_SPLIT", raising=False)
    n_tiled = sum(spec.tile_plan(s)["tiled"] for s in range(8))
    assert n_tiled >= 4 if tiling == "auto" else n_tiled == 0
    rng = np.random.default_rng(N + 1)
    spec.state_init()
    full.state_init()
    prefix = 0
    for s in range(8):
        p = spec.stage_probs(s, prefix)
        assert p == full.stage_probs(s, prefix), s
        if s + 1 == 8:
            break
        b = s & 1 if s < 4 else int(rng.integers(2))
        if min(p) <= 1e-300:
            b = int(p[1] > p[0])
        spec.stage_collapse(b, p[b])
        full.stage_collapse(b, p[b])
        for first in [0, N - 4096] + [int(x) for x in rng.integers(0, N - 4096, 4)]:
            for x in (0, 1):
                assert np.array_equal(arr(spec.state_read(x, first, 4096)),
                                      arr(full.state_read(x, first, 4096))), (s, first)
        prefix |= b << s
    for idx in range(3):
        r, q = spec.run(11, idx), full.run(11, idx)
        assert r.bits.j == q.bits.j and [x.p1 for x in r.trace] == [x.p1 for x in q.trace], idx


@pytest.mark.parametrize("N,a", [(16777207, 2), (268435247, 3), (4194301, 7), (268435247, 5)])
def test_small_multiplier_streams_vs_gather(cuda_ok, N, a):
    """The last stages (multipliers a, a^2, a^4 ... <= 1024) stage their A
    gathered runs through shared memory (kSrcStreams, from the run start e_1 and
    from a general state), or, for 512 <= A with more than 2^18 A-long rows
    (N = 268435247, A = 625: the config-4 case), run as tiles of the consecutive
    rows j A (tile_plan.hpp make_small_a_plan): bit-identical to the
    per-amplitude gather."""
    rng = np.random.default_rng(N + a)
    fast, ref = engine(N, a), engine(N, a, tiling="off")
    pows = fast.stage_multipliers()
    s0 = fast.t - 6
    assert sum(1 for s in range(s0, fast.t) if 1 < pows[s] <= 1024) >= 2
    for s in range(s0, fast.t):
        if 512 <= pows[s] and N // pows[s] > (1 << 18):
            pl = fast.tile_plan(s)
            assert pl["tiled"] and pl["H"] == N // pows[s] and pl["u"] == 1, pl
    fast.state_init()
    ref.state_init()
    prefix = 0
    for s in range(s0, fast.t):
        p = fast.stage_probs(s, prefix)
        assert p == ref.stage_probs(s, prefix), s
        d0, d1 = fast.block_sums()
        e0, e1 = ref.block_sums()
        assert np.array_equal(d0, e0) and np.array_equal(d1, e1), s
        if s + 1 == fast.t:
            break
        b = int(rng.integers(2)) if min(p) > 1e-300 else int(p[1] > p[0])
        fast.stage_collapse(b, p[b])
        ref.stage_collapse(b, p[b])
        for first in [0, N - 4096] + [int(x) for x in rng.integers(0, N - 4096, 6)]:
            for x in (0, 1):
                assert np.array_equal(arr(fast.state_read(x, first, 4096)),
                                      arr(ref.state_read(x, first, 4096))), (s, first)
        prefix |= b << s


# ------------------------------------------------- full-size properties
def test_c3_size_run_properties(cuda_ok, oracle):
    """N = 16777207 (config 3): first stages match the oracle exactly; the full
    run keeps the norm (check_norms) and is replayable (same seed -> same bits)."""
    N, a, t = 16777207, 1234567, 48
    eng = engine(N, a, t)
    r1 = eng.run(11, 0)
    r2 = eng.run(11, 0)
    assert r1.bits.j == r2.bits.j and [x.p1 for x in r1.trace] == [x.p1 for x in r2.trace]
    orc = oracle.engine(N, a, N.bit_length(), t)
    orc.state_init()
    eng.state_init()
    prefix = 0
    for s in range(3):
        q0, q1 = orc.stage_probs(s, prefix, 1)
        p0, p1 = eng.stage_probs(s, prefix)
        assert (p0, p1) == (q0, q1)
        b = r1.trace[s].observed_bit
        orc.collapse(b, q1 if b else q0)
        eng.stage_collapse(b, p1 if b else p0)
        prefix |= b << s


@pytest.mark.slow
def test_c4_size_stages(cuda_ok):
    """N = 4294967213 (config 4, 2 x 68.7 GB on one GPU): stage masses stay
    normalised and the index map is exact at both ends of the range."""
    N, a = 4294967213, 3
    eng = engine(N, a, 64)
    a_pows = eng.stage_multipliers()
    eng.state_init()
    prefix = 0
    for s in range(4):
        p0, p1 = eng.stage_probs(s, prefix)
        assert abs(p0 + p1 - 1.0) < 1e-12
        b = 1 if p1 >= p0 else 0
        eng.stage_collapse(b, p1 if b else p0)
        prefix |= b << s
    from oracle import Oracle
    o = Oracle()
    inv = o.mod_inverse(a_pows[5], N)
    got = list(eng.index_map(5, N - 2048, 2048))
    assert got == [(inv * z) % N for z in range(N - 2048, N)]


def test_tile_plans_partition_and_auto_selection(cuda_ok):
    """AUTO tiles every non-identity stage of the bench problems that has a plan
    (at these sizes every plan has >= 16 chunks per CTA, whatever its band
    count); rows of every plan satisfy the three-gap partition (checked
    exhaustively at small N)."""
    for N, a in [(4294967213, 5), (268435247, 3), (16777207, 2)]:
        eng = engine(N, a)
        forced = engine(N, a, tiling="force")
        pows = eng.stage_multipliers()
        ntiled = 0
        for s in range(1, eng.t):
            pl = eng.tile_plan(s)
            if N == 4294967213 and pows[s] > 1 << 20:  # config 4: every "random" multiplier tiles
                assert pl["tiled"], (N, s, pl)
            assert pl == forced.tile_plan(s), (N, s)
            if pl["tiled"]:
                ntiled += 1
                H = pl["H"]
                if pl["u"] == 1 and H == N // pows[s] and H > (1 << 18):
                    # small-multiplier plan: the A-long runs j A, the last one A + N mod A
                    A = pows[s]
                    assert 512 <= A and pl["du"] == A and pl["dv"] == A + N % A
                    assert pl["v"] == H - 1 and (H - 1) * A + pl["dv"] == N
                    continue
                assert pl["du"] >= 512 and pl["dv"] >= 512 and H <= N // 640
                assert pl["du"] + pl["dv"] <= 3 * (N // H + 1) and H >= 256
        assert ntiled >= eng.t - 6, (N, ntiled)  # all but stage 0 and the tiny multipliers
    N, a = 1048351, 12345
    eng = engine(N, a, 8, tiling="force")
    pows = eng.stage_multipliers()
    ntiled = 0
    for s in range(1, 8):
        pl = eng.tile_plan(s)
        if not pl["tiled"]:
            continue
        ntiled += 1
        H, u, v, du, dv, A = pl["H"], pl["u"], pl["v"], pl["du"], pl["dv"], pows[s]
        cover = np.zeros(N, dtype=np.int8)
        for j in range(H):
            L = du if j + u < H else (dv if j >= v else du + dv)
            z = j * A % N
            assert z + L <= N
            cover[z:z + L] += 1
        assert cover.min() == 1 and cover.max() == 1
    assert ntiled >= 5
