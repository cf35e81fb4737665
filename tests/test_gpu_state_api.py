"""The reference's per-gate API on the device-resident
ShardedState (csrc/sv.cu) against the UNMODIFIED reference's own per-gate
functions (oracle/_ref through ref_shim: init_state, apply_oracle, apply_phase,
apply_hadamard_top, group_norm_squared, reset_top, build_permutation_plan):
every amplitude after every gate bit-identical, norms bit-identical, errors as
the reference raises them; and the pins of the reference's own test file
(proj/tests/test_statevector.cpp:25-59 composed run == engine,
:77-119 the Fig.-3 exchange plan, :121-151 oracle examples and inverse
restoration)."""
import math
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

K = 1.0 / math.sqrt(2.0)


def E(kind="none", delta=0.0, pauli=None):
    from paper_2308_05047_b200 import ErrorConfig, ErrorKind, PauliProbs
    return ErrorConfig(ErrorKind[kind], delta, PauliProbs(*pauli) if pauli else None)


def reinit(err):
    """reinit_state (noise.cpp:89-95) through the reference"""
    import ctypes as C
    from oracle import Oracle, make_error
    o = Oracle()
    w = (C.c_double * 4)()
    p = err.pauli
    o.lib.so_reinit_state(C.byref(make_error(err.kind.name, err.delta, p.px if p else 0.0,
                                             p.py if p else 0.0, p.pz if p else 0.0)), w)
    return (complex(w[0], w[1]), complex(w[2], w[3]))


def same_state(st, ref, n):
    g = 1 << (n - 1)
    got = st.read_array(0, 1 << n)
    want = np.array(ref.read_group(0, 0, g) + ref.read_group(1, 0, g))
    assert np.array_equal(got, want)


def test_gates_bit_identical_to_reference(cuda_ok, reference):
    import paper_2308_05047_b200 as shs
    from oracle import make_error
    rng = random.Random(3)
    for N, a, t, kind, delta in [(4087, 1001, 12, "phase_init", 0.3), (55, 16, 8, "none", 0.0),
                                 (65521, 17, 10, "amplitude_init", 0.15),
                                 (1048351, 12345, 6, "none", 0.0)]:
        n = N.bit_length() + 1
        err = E(kind, delta)
        st = shs.init_state(n, reinit(err), 4)
        ref = reference.state(n, make_error(kind, delta), 4)
        same_state(st, ref, n)
        pows = [0] * t
        pows[t - 1] = a % N
        for s in range(t - 1, 0, -1):
            pows[s - 1] = pows[s] * pows[s] % N
        prefix = 0
        for s in range(t):
            shs.apply_oracle(st, pows[s], N)
            ref.oracle(pows[s], N)
            shs.apply_phase(st, s, prefix)
            ref.phase(s, prefix)
            shs.apply_hadamard_top(st)
            ref.hadamard()
            same_state(st, ref, n)
            p0, p1 = st.group_norms()
            assert (p0, p1) == (ref.group_norm(0), ref.group_norm(1))
            b = rng.randrange(2) if min(p0, p1) > 1e-6 else int(p1 > p0)
            eb = rng.random() < 0.2 and min(p0, p1) > 1e-6
            src = 1 - b if eb else b
            ps = p1 if src else p0
            shs.reset_top(st, b, eb, reinit(err), ps)
            ref.reset(b, eb, ps)
            same_state(st, ref, n)
            prefix |= b << s
        st.close()


def test_measure_and_reset_errors(cuda_ok):
    import paper_2308_05047_b200 as shs
    zero = shs.init_state(4, (1.0, 0.0), 2)
    for i in range(20):
        m = shs.measure_top(zero, 1, i, 0, E())
        assert m["p1"] == 0.0 and m["sampled_bit"] == 0
    st = shs.init_state(4, (1.0, 0.0), 2)  # |0>|1>; test_statevector.cpp:223-232
    shs.reset_top(st, 0, False, (K, K), 1.0)
    assert st.amp_xy(0, 1) == complex(K, 0.0) and st.amp_xy(1, 1) == complex(K, 0.0)
    assert abs(st.norm_squared() - 1.0) < 1e-9
    with pytest.raises(shs.DegenerateBranchError):
        shs.reset_top(st, 1, True, (K, K), 0.0)
    with pytest.raises(ValueError):
        shs.ShardedState(7, 3)
    with pytest.raises(ValueError):
        shs.ShardedState(3, 8)
    with pytest.raises(shs.NotInvertibleError):
        shs.apply_oracle(shs.ShardedState(7, 4), 5, 55)


def test_exchange_plan_fig3_and_reference(cuda_ok, reference):
    """test_statevector.cpp:77-119 (N = 55, a = 16, n = 7, 16 shards), plus the
    gather and pair counts against the reference's own build_permutation_plan."""
    import paper_2308_05047_b200 as shs
    layout = shs.make_shard_layout(7, 16)
    plan = shs.build_permutation_plan(16, 55, layout)
    assert plan.y_limit == 55 and not plan.identity
    assert sorted(plan.gather) == list(range(55))
    assert plan.gather[48] == 3
    assert sum(sum(r) for r in plan.pair_counts) == 55
    assert all(plan.pair_counts[s][7] == 0 for s in range(8))
    assert shs.plan_receive_lists(plan, 7) == []
    inv = shs.build_permutation_plan(plan.a_inv, 55, layout)
    assert all(inv.gather[plan.gather[z]] == z for z in range(55))
    ident = shs.build_permutation_plan(1, 55, layout)
    assert ident.identity and ident.gather == list(range(55))
    for xr in range(8):
        recv = sum(len(x.local_index) for x in shs.plan_receive_lists(plan, xr))
        z0 = xr * layout.shard_size()
        assert recv == (0 if z0 >= 55 else min(55 - z0, layout.shard_size()))
    rng = random.Random(9)
    for _ in range(12):
        N = rng.randrange(3, 1 << 16)
        a = rng.randrange(1, N)
        if math.gcd(a, N) != 1:
            continue
        n = N.bit_length() + 1
        shards = 1 << rng.randrange(1, min(n - 1, 6) + 1)
        want = reference.plan(a, N, n, shards)
        got = shs.build_permutation_plan(a, N, shs.make_shard_layout(n, shards))
        assert got.gather == want["gather"] and got.a_inv == want["a_inv"]
        assert got.pair_counts == want["pair_counts"] and got.identity == want["identity"]
        lay = got.layout
        shard = lay.shard_size()
        for xr in range(lay.group_shards()):  # lists from the reference's definitions
            z0, z1 = xr * shard, min(got.y_limit, (xr + 1) * shard)
            rl = {}
            for z in range(z0, max(z0, z1)):
                rl.setdefault(want["gather"][z] >> (lay.n - lay.g), []).append(z - z0)
            assert [(x.xrank, x.local_index) for x in shs.plan_receive_lists(got, xr)] == \
                sorted(rl.items())
            sl = {}
            for z in range(got.y_limit):
                src = want["gather"][z]
                if src >> (lay.n - lay.g) == xr:
                    sl.setdefault(z >> (lay.n - lay.g), []).append(src - xr * shard)
            assert [(x.xrank, x.local_index) for x in shs.plan_send_lists(got, xr)] == \
                sorted(sl.items())


def test_oracle_examples_and_inverse_restoration(cuda_ok):
    """test_statevector.cpp:121-151"""
    import paper_2308_05047_b200 as shs
    st = shs.init_state(7, (K, K), 4)
    st.set_amp(st.group_base(1) + 3, complex(0.5, 0.25))
    shs.apply_oracle(st, 16, 55)
    assert st.amp_xy(1, 48) == complex(0.5, 0.25)
    assert st.amp_xy(1, 3) == 0
    assert st.amp_xy(0, 1) == complex(K, 0)
    st.set_amp(st.group_base(1) + 60, complex(0.125, 0.0))
    shs.apply_oracle(st, 16, 55)
    assert st.amp_xy(1, 60) == complex(0.125, 0.0)
    rng = random.Random(17)
    for _ in range(40):
        n_mod = 3 + rng.randrange((1 << 16) - 3)
        a = 2 + rng.randrange(n_mod - 2)
        if math.gcd(a, n_mod) != 1:
            continue
        n = n_mod.bit_length() + 1
        s = shs.ShardedState(n, 4)
        vals = [complex(rng.random() - 0.5, rng.random() - 0.5) for _ in range(min(n_mod, 64))]
        s.write(s.group_base(1), vals)
        before = s.copy()
        shs.apply_oracle(s, a, n_mod)
        shs.apply_oracle(s, pow(a, -1, n_mod), n_mod)
        assert np.array_equal(s.read_array(0, 1 << n), before.read_array(0, 1 << n))


def test_composed_run_equals_engine(cuda_ok):
    """test_statevector.cpp:25-59 + 236-279: the run assembled from the device
    per-gate API equals the fused engine bit for bit (6 error models)."""
    import paper_2308_05047_b200 as shs
    errs = [E(), E("classical_measure", 0.2), E("amplitude_init", 0.15), E("phase_init", 0.3),
            E("bitflip", 0.1), E("quantum_measure", 0.03, (0.02, 0.01, 0.05))]
    for err in errs:
        for N, a in [(15, 7), (21, 11), (55, 16), (57, 20)]:
            prob = shs.FactoringProblem.make(N, a, 10)
            eng = shs.IterativeShorEngine(prob, err, shs.SimulatorOptions(shard_count=4))
            pows = eng.stage_multipliers()
            w = reinit(err)
            for idx in range(4):
                fused = eng.run(31, idx)
                st = shs.init_state(prob.L + 1, w, 4)
                observed = sampled = 0
                trace = []
                for s in range(prob.t):
                    shs.apply_oracle(st, pows[s], N)
                    shs.apply_phase(st, s, observed)
                    shs.apply_hadamard_top(st)
                    m = shs.measure_top(st, 31, idx, s, err)
                    trace.append((m["p1"], m["sampled_bit"], m["observed_bit"]))
                    observed |= m["observed_bit"] << s
                    sampled |= m["sampled_bit"] << s
                    if s + 1 < prob.t:
                        src = 1 - m["sampled_bit"] if m["error_branch"] else m["sampled_bit"]
                        shs.reset_top(st, m["sampled_bit"], m["error_branch"], w,
                                      st.group_norm_squared(src))
                assert [(x.p1, x.sampled_bit, x.observed_bit) for x in fused.trace] == trace
                assert fused.j_sampled == sampled
                st.close()
