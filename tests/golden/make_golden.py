"""Generate tests/golden/*.json from the UNMODIFIED reference library.

Run in the dev container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

It loads oracle/_ref/libshorsim_ref.so (built from /root/reference/proj/src by
oracle/Makefile) and records the reference's own outputs for the hot-path
pins of SURVEY.md §4 / §8c. Floats are stored as hex strings (float.hex) so
fixtures are bit-exact. The GPU box never runs this script.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference, make_error  # noqa: E402

ERRORS = {
    "none": dict(kind="none"),
    "classical_measure": dict(kind="classical_measure", delta=0.2),
    "amplitude_init": dict(kind="amplitude_init", delta=0.15),
    "phase_init": dict(kind="phase_init", delta=0.3),
    "bitflip": dict(kind="bitflip", delta=0.1),
    "quantum_measure": dict(kind="quantum_measure", delta=0.03, px=0.02, py=0.01, pz=0.05),
}


def hexlist(xs):
    return [float(x).hex() for x in xs]


def run_record(eng, seed, idx):
    r = eng.run(seed, idx)
    r["p1"] = hexlist(r["p1"])
    r["j"] = str(r["j"])
    r["j_sampled"] = str(r["j_sampled"])
    return r


def main():
    ref = Reference()
    out = {}

    # 1. Philox KAT, proj/tests/test_util.cpp:82-89, plus addressed draws
    out["philox"] = {
        "kat": {"key": 0, "ctr": [0, 0, 0, 0], "out": ref.philox(0, [0, 0, 0, 0])},
        "vectors": [{"key": k, "ctr": c, "out": ref.philox(k, c)}
                    for k, c in [(42, [1, 2, 3, 0]), (2**64 - 1, [2**32 - 1, 7, 9, 1]),
                                 (31, [0, 5, 9, 0]), (123456789, [17, 0, 0, 1])]],
    }

    # 2. Fig.-3 exchange plan, proj/tests/test_statevector.cpp:77-119
    plan = ref.plan(16, 55, 7, 16)
    out["plan_fig3"] = {"a_pow": 16, "N": 55, "n": 7, "shards": 16, **plan}
    out["plans"] = []
    for a_pow, N in [(4, 15), (7, 15), (11, 21), (1001, 4087), (2024, 8051), (12345, 1048351)]:
        n = N.bit_length() + 1
        p = ref.plan(a_pow, N, n, 4)
        out["plans"].append({"a_pow": a_pow, "N": N, "n": n, "a_inv": p["a_inv"],
                             "head": p["gather"][:64], "tail": p["gather"][-64:],
                             "checksum": sum((i + 1) * g for i, g in enumerate(p["gather"]))
                             % (2**61 - 1)})

    # 3. multipliers, proj/tests/test_statevector.cpp:327-336
    e = ref.engine(15, 7, 4, 8)
    out["multipliers_15_7"] = e.multipliers()

    # 4. engine == composed ops pin set, proj/tests/test_statevector.cpp:236-279
    runs = []
    for ename, ekw in ERRORS.items():
        err = make_error(**ekw)
        for N, a in [(15, 7), (21, 11), (55, 16), (57, 20)]:
            eng = ref.engine(N, a, N.bit_length(), 10, err)
            for idx in range(8):
                runs.append({"error": ename, "N": N, "a": a, "t": 10, "seed": 31, "idx": idx,
                             **run_record(eng, 31, idx)})
    out["engine_runs"] = runs

    # 5. byte-stability cases, test_harness.cpp:177-195 and acceptance criterion 10
    eng = ref.engine(4087, 1001, 12, 24)
    out["run_4087"] = [{"seed": 7, "idx": 3, **run_record(eng, 7, 3)}] + \
        [{"seed": 3, "idx": i, **run_record(eng, 3, i)} for i in range(4)]
    eng = ref.engine(8051, 2024, 13, 26)
    out["run_8051"] = [{"seed": 9, "idx": i, **run_record(eng, 9, i)} for i in range(32)]

    # 6. acceptance c2 prefix: N=15, a=7, t=8, seed 2, idx 0..63
    eng = ref.engine(15, 7, 4, 8)
    out["run_15_c2"] = [{"seed": 2, "idx": i, **run_record(eng, 2, i)} for i in range(64)]

    # 7. forced sequence amplitude dumps via the per-gate API (CS3), N=55, a=16, t=6
    forced = []
    for ename in ["none", "phase_init", "amplitude_init"]:
        err = make_error(**ERRORS[ename])
        N, a, t = 55, 16, 6
        n = N.bit_length() + 1
        st = ref.state(n, err, 4)
        a_pows = [0] * t
        a_pows[t - 1] = a % N
        for s in range(t - 1, 0, -1):
            a_pows[s - 1] = a_pows[s] * a_pows[s] % N
        bits = [1, 0, 1, 1, 0, 1]
        prefix = 0
        steps = []
        for s in range(t):
            st.oracle(a_pows[s], N)
            st.phase(s, prefix)
            st.hadamard()
            p1 = st.group_norm(1)
            p0 = st.group_norm(0)
            post = {"g0": hexlist(st.read_group(0, 0, 64)), "g1": hexlist(st.read_group(1, 0, 64))}
            b = bits[s]
            p_src = p1 if b else p0
            rec = {"s": s, "p0": float(p0).hex(), "p1": float(p1).hex(), "bit": b, "post_h": post}
            if p_src > 1e-300 and s + 1 < t:
                st.reset(b, False, p_src)
                rec["post_reset"] = {"g0": hexlist(st.read_group(0, 0, 64)),
                                     "g1": hexlist(st.read_group(1, 0, 64))}
            prefix |= b << s
            steps.append(rec)
        forced.append({"error": ename, "N": N, "a": a, "t": t, "bits": bits, "steps": steps})
    out["forced"] = forced

    # 8. exhaustive distribution, test_statevector.cpp:357-364
    dist = ref.exhaustive(15, 7, 4, 8)
    out["exhaustive_15_7_8"] = hexlist(dist)
    # error-model marginalisation, test_statevector.cpp:366-396 and test_noise.cpp:100-116
    ex = []
    for N, a, t, ename, ekw in [(15, 7, 5, "classical", dict(kind="classical_measure", delta=0.3)),
                                (15, 7, 5, "quantum", dict(kind="quantum_measure", delta=0.1, px=0.05, py=0.05, pz=0.1)),
                                (21, 2, 8, "pz_only", dict(kind="quantum_measure", delta=0.0, px=0.0, py=0.0, pz=0.3)),
                                (55, 16, 8, "none", dict(kind="none")),
                                (35, 4, 7, "bitflip", dict(kind="bitflip", delta=0.05)),
                                (57, 5, 6, "phase", dict(kind="phase_init", delta=0.2)),
                                (33, 5, 6, "amplitude", dict(kind="amplitude_init", delta=0.1))]:
        d = ref.exhaustive(N, a, N.bit_length(), t, make_error(**ekw))
        ex.append({"N": N, "a": a, "t": t, "name": ename, "error": ekw, "dist": hexlist(d)})
    out["exhaustive_cases"] = ex

    out["_meta"] = {"generator": "tests/golden/make_golden.py",
                    "reference": "/root/reference/proj (unmodified), oracle/_ref/libshorsim_ref.so",
                    "errors": ERRORS}
    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
