"""The reference's OWN callers, compiled unchanged from /root/reference, linked
against the B200 engine (oracle/b200_link.cpp defines IterativeShorEngine's
constructor and run() over the C ABI): simulate_to_jsonl output must be
byte-identical to the reference engine's, and the acceptance criteria that use
the engine must pass. Binaries are built by build() where /root/reference
exists and travel to the GPU box."""
import os
import subprocess

import pytest

from oracle import (ACCEPTANCE_B200, ACCEPTANCE_REF, DROPIN_TESTS, SIMULATE_B200, SIMULATE_DROPIN,
                    SIMULATE_REF)

need = pytest.mark.skipif(not (os.path.exists(SIMULATE_REF) and os.path.exists(SIMULATE_B200)),
                          reason="drop-in binaries not built (need /root/reference at build time)")

CASES = [
    # proj/tests/test_harness.cpp:177-195 and acceptance criterion 10 problems
    ("4087", "1001", "24", "4", "3", "2", None),
    ("8051", "2024", "26", "32", "9", "16", None),
    ("15", "7", "8", "64", "2", "4", None),
    ("4087", "1001", "24", "8", "5", "4", "kind=quantum_measure,px=0.02,py=0.01,pz=0.05"),
    ("4087", "1001", "24", "8", "5", "4", "kind=classical_measure,delta=0.2"),
    ("4087", "1001", "24", "8", "5", "4", "kind=phase_init,delta=0.3"),
    ("4087", "1001", "24", "8", "5", "4", "kind=amplitude_init,delta=0.15"),
    ("4087", "1001", "24", "8", "5", "4", "kind=bitflip,delta=0.1"),
    ("262139", "31337", "12", "4", "1", "4", None),
]


def run(exe, args, timeout=600):
    return subprocess.run([exe] + list(args), capture_output=True, text=True, timeout=timeout)


@need
def test_reference_simulate_runs_on_cpu():
    r = run(SIMULATE_REF, ["15", "7", "8", "2", "2"])
    assert r.returncode == 0 and '"schema":"shorsim/simulate"' in r.stdout


@need
def test_b200_link_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    r = run(SIMULATE_B200, ["15", "7", "8", "2", "2"])
    assert r.returncode != 0 and "cuda" in r.stderr.lower()


@need
@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(x for x in c[:5]) + ("-" + c[6].split(",")[0][5:] if c[6] else ""))
def test_simulate_jsonl_byte_identical(cuda_ok, case):
    args = [x for x in case if x is not None]
    ref = run(SIMULATE_REF, args)
    ours = run(SIMULATE_B200, args)
    assert ref.returncode == 0, ref.stderr
    assert ours.returncode == 0, ours.stderr
    assert ours.stdout == ref.stdout


@need
@pytest.mark.gpu
@pytest.mark.parametrize("case", [CASES[0], CASES[3], CASES[8]], ids=["4087", "4087-quantum", "262139"])
def test_simulate_jsonl_byte_identical_over_virtual_shards(cuda_ok, case):
    """Row N1: the reference's unchanged harness with the engine sharded over
    devices (SHS_DEVICES=0,0: two shards on this GPU) — byte-identical JSONL."""
    args = [x for x in case if x is not None]
    ref = run(SIMULATE_REF, args)
    env = dict(os.environ, SHS_DEVICES="0,0")
    ours = subprocess.run([SIMULATE_B200] + args, capture_output=True, text=True, timeout=600,
                          env=env)
    assert ref.returncode == 0, ref.stderr
    assert ours.returncode == 0, ours.stderr
    assert ours.stdout == ref.stdout


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ACCEPTANCE_B200), reason="not built")
@pytest.mark.parametrize("criterion", ["1", "2", "10"])
def test_reference_acceptance_criteria_on_b200(cuda_ok, criterion):
    r = run(ACCEPTANCE_B200, ["--criterion", criterion], timeout=1200)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert f"CRITERION {criterion}: PASS" in r.stdout


# ---- the drop-in header (include/dropin/shorsim/statevector.hpp): the
# reference's callers and unit tests compiled UNCHANGED against it (no
# proj/src/statevector.cpp linked), with a doctest-compatible shim
@pytest.mark.gpu
@pytest.mark.parametrize("name", ["statevector", "noise", "harness"])
def test_reference_unit_tests_against_dropin_header(cuda_ok, name):
    exe = DROPIN_TESTS[name]
    if not os.path.exists(exe):
        pytest.skip("not built")
    r = run(exe, [], timeout=1800)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed |" in r.stdout


@need
@pytest.mark.gpu
@pytest.mark.parametrize("case", [CASES[0], CASES[1], CASES[4], CASES[8]],
                         ids=["4087", "8051", "4087-classical", "262139"])
def test_simulate_jsonl_byte_identical_dropin_header(cuda_ok, case):
    if not os.path.exists(SIMULATE_DROPIN):
        pytest.skip("not built")
    args = [x for x in case if x is not None]
    ref = run(SIMULATE_REF, args)
    ours = run(SIMULATE_DROPIN, args)
    assert ref.returncode == 0 and ours.returncode == 0, ours.stderr
    assert ours.stdout == ref.stdout
