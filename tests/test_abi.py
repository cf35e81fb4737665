"""The drop-in boundary on the CPU: libshorsim_b200.so loads, exports every
symbol include/shorsim_b200.h declares, validates exactly like the reference
(errors raised before any device call), never falls back to the CPU, and its
host-side scalar model (sampling / error hooks) equals the oracle's."""
import os
import random
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shorsim_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(shs_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2308_05047_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    declared = {name for name, _, _ in _lib.SIGNATURES}
    assert declared == set(syms)


def test_build_info_names_sm100a():
    from paper_2308_05047_b200 import build_info
    assert "sm_100a" in build_info()


def _mk(N, a, t=None, err=None, **opt):
    from paper_2308_05047_b200 import (ErrorConfig, FactoringProblem, IterativeShorEngine,
                                       SimulatorOptions)
    return IterativeShorEngine(FactoringProblem.make(N, a, t), err or ErrorConfig(),
                               SimulatorOptions(**opt))


def test_validation_matches_reference_order():
    import paper_2308_05047_b200 as shs
    E = shs.ErrorConfig
    K = shs.ErrorKind
    with pytest.raises(shs.ConfigError):  # ErrorConfig::validate first (statevector.cpp:289)
        _mk(15, 7, err=E(K.bitflip, 1.5), qubit_ceiling=3)
    with pytest.raises(shs.ConfigError):
        _mk(15, 7, err=E(K.quantum_measure, 0.1))  # missing Pauli triple
    with pytest.raises(shs.ConfigError):
        _mk(15, 7, err=E(K.classical_measure, 0.1, shs.PauliProbs(0.1, 0, 0)))
    with pytest.raises(shs.CeilingExceededError):  # statevector.cpp:291-294
        _mk(4087, 1001, 24, qubit_ceiling=12)
    for shards in (0, 1, 3, 6):  # make_shard_layout, statevector.cpp:67-68
        with pytest.raises(ValueError):
            _mk(15, 7, shard_count=shards)
    with pytest.raises(ValueError):  # more shards than group states (:70)
        _mk(15, 7, shard_count=32)
    with pytest.raises(shs.NotInvertibleError) as ei:  # mod_inverse, numtheory.cpp:39-46
        _mk(15, 6, 8)
    assert ei.value.gcd == 3


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2308_05047_b200 as shs
    with pytest.raises(shs.CudaError):
        _mk(15, 7, 8)


def test_host_sampling_equals_oracle(oracle):
    import paper_2308_05047_b200 as shs
    from oracle import make_error
    cases = [(shs.ErrorConfig(), make_error()),
             (shs.ErrorConfig(shs.ErrorKind.classical_measure, 0.3),
              make_error("classical_measure", 0.3)),
             (shs.ErrorConfig(shs.ErrorKind.quantum_measure, 0.1, shs.PauliProbs(0.05, 0.05, 0.1)),
              make_error("quantum_measure", 0.1, 0.05, 0.05, 0.1))]
    rng = random.Random(9)
    for e, oe in cases:
        for _ in range(500):
            p1 = rng.choice([0.0, 1.0, 0.5, rng.random()])
            seed, idx, st = rng.getrandbits(64), rng.getrandbits(32), rng.randrange(128)
            m = shs.sample_measurement(p1, seed, idx, st, e)
            o = oracle.sample(p1, seed, idx, st, oe)
            assert (m["sampled_bit"], m["observed_bit"], int(m["error_branch"]),
                    int(m["classical_flip"])) == tuple(o)


def test_parse_error_config_grammar():
    import paper_2308_05047_b200 as shs
    c = shs.parse_error_config("kind=quantum_measure,px=0.005,py=0.005")
    assert c.kind == shs.ErrorKind.quantum_measure and abs(c.delta - 0.01) < 1e-15
    assert c.pauli.pz == 0.0
    c = shs.parse_error_config("kind=amplitude_init,delta=0.1")
    assert c.kind == shs.ErrorKind.amplitude_init and c.delta == 0.1
    assert shs.parse_error_config("kind=none").kind == shs.ErrorKind.none
    for bad in ["kind=bitflip", "kind=foo,delta=0.1", "delta=0.1", "kind=none,zz=1",
                "kind=quantum_measure,px=0.1", "kind=bitflip,delta=2",
                "kind=quantum_measure,px=0.1,py=0.1,delta=0.5", "garbage"]:
        with pytest.raises(shs.ConfigError):
            shs.parse_error_config(bad)


def test_recommended_t_and_problem():
    import paper_2308_05047_b200 as shs
    assert shs.recommended_t(15) == 8
    assert shs.recommended_t(4294967213) == 64
    assert shs.recommended_t(34359737977) == 70
    p = shs.FactoringProblem.make(16777207, 3)
    assert (p.L, p.t, p.qubits()) == (24, 48, 25)
