"""Host-side logic of the sharded engine on CPU: exact digit combine, and the
product driver (ShardedShorEngine + DistGroup) running across 2 gloo processes
with numpy shards (tests/cpu_shard.py), bit-identical to the oracle's
single-process run with the exact combine."""
import math
import os
import random
import socket
from fractions import Fraction

import pytest
import torch.multiprocessing as mp

from cpu_shard import exact_digits

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_digits_to_probs_is_correctly_rounded():
    from paper_2308_05047_b200 import digits_to_probs
    rng = random.Random(1)
    for _ in range(100):
        k = rng.randrange(1, 200)
        v0 = [rng.random() * 2.0 ** rng.randrange(-70, 0) for _ in range(k)]
        v1 = [rng.random() * 2.0 ** rng.randrange(-70, 0) for _ in range(k)]
        # split over 3 "shards" and sum their digits, as the allreduce does
        parts = [exact_digits(v0[i::3]) + exact_digits(v1[i::3]) for i in range(3)]
        total = [sum(x) for x in zip(*parts)]
        p0, p1 = digits_to_probs(total)
        assert p0 == float(sum(Fraction(x) for x in v0))
        assert p1 == float(sum(Fraction(x) for x in v1))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [  # (N, a, t, error kind, delta, pauli)
    (262139, 31337, 10, "none", 0.0, None),
    (100003, 777, 9, "phase_init", 0.2, None),
    (65537 * 3, 101, 8, "quantum_measure", 0.02, (0.01, 0.01, 0.0)),
    (8051, 2024, 12, "bitflip", 0.05, None),
]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import paper_2308_05047_b200 as shs
    from cpu_shard import CpuShard
    from oracle import Oracle, make_error

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        _run_cases(rank, world, dist, q)
    except Exception as exc:  # report instead of leaving the peer blocked
        q.put((rank, f"{type(exc).__name__}: {exc}"))
    finally:
        dist.destroy_process_group()


def _run_cases(rank, world, dist, q):
    import paper_2308_05047_b200 as shs
    from cpu_shard import CpuShard
    from oracle import Oracle, make_error
    if True:
        orc = Oracle()
        results = []
        for N, a, t, kind, delta, pauli in CASES:
            err = shs.ErrorConfig(shs.ErrorKind[kind], delta,
                                  shs.PauliProbs(*pauli) if pauli else None)
            oe = make_error(kind, delta, *(pauli or (0.0, 0.0, 0.0)))
            w = [0.0] * 4
            import ctypes as C
            warr = (C.c_double * 4)()
            orc.lib.so_reinit_state(C.byref(oe), warr)
            w = tuple(warr)
            prob = shs.FactoringProblem.make(N, a, t)
            shard = CpuShard(N, a, t, w, rank, world, dist)
            eng = shs.ShardedShorEngine(prob, err, shs.SimulatorOptions(qubit_ceiling=64), [shard],
                                        shs.DistGroup(shard, attach_ipc=False))
            ref = orc.engine(N, a, N.bit_length(), t, oe)
            for idx in range(2):
                r = eng.run_stepwise(17, idx)
                o = ref.run(17, idx, 1)  # oracle with the exact combine
                results.append((N, idx, r.bits.j == o["j"], [x.p1 for x in r.trace] == o["p1"],
                                r.j_sampled == o["j_sampled"]))
        q.put((rank, results))


def test_sharded_driver_two_gloo_ranks_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        rank, res = q.get(timeout=300)
        assert not isinstance(res, str), res
        out[rank] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]
    for N, idx, bits_ok, p1_ok, js_ok in out[0]:
        assert bits_ok and p1_ok and js_ok, (N, idx)


def test_too_many_shards_is_rejected():
    import paper_2308_05047_b200 as shs
    with pytest.raises(ValueError):
        shs.Shard(shs.FactoringProblem.make(15, 7, 8), shs.ErrorConfig(),
                  shs.SimulatorOptions(qubit_ceiling=64), 1, 2)


def _barrier_worker(rank, parties, name, rounds, path, q):
    import ctypes as C
    import sys
    sys.path.insert(0, ROOT)
    from paper_2308_05047_b200 import _lib as L
    lib = L.load()
    h = C.c_void_p()
    try:
        assert lib.shs_node_barrier_open(name.encode(), parties, 1 if rank == 0 else 0,
                                         C.byref(h)) == 0
        seen = []
        for r in range(rounds):
            # phase A: everyone appends "r", barrier, everyone checks all parties wrote r
            with open(path, "a") as f:
                f.write(f"{rank}:{r}\n")
            assert lib.shs_node_barrier_arrive(h) == 0
            lines = open(path).read().split()
            seen.append(sum(1 for x in lines if x.endswith(f":{r}")))
            assert lib.shs_node_barrier_arrive(h) == 0  # nobody starts r+1 before all checked r
        q.put((rank, seen))
    except Exception as exc:
        q.put((rank, f"{type(exc).__name__}: {exc}"))
    finally:
        if h:
            lib.shs_node_barrier_close(h)


def test_node_barrier_orders_processes(tmp_path):
    """The host barrier of multi-process sharded runs (shs_shards_run): with 3
    processes, every process sees every party's write of round r after the
    barrier, and nobody's write of round r+1 before the second barrier."""
    import uuid
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    parties, rounds = 3, 40
    name = f"/shs_test_{uuid.uuid4().hex[:12]}"
    path = str(tmp_path / "log.txt")
    open(path, "w").close()
    procs = [ctx.Process(target=_barrier_worker, args=(r, parties, name, rounds, path, q))
             for r in range(parties)]
    for p in procs:
        p.start()
    out = {}
    for _ in procs:
        rank, res = q.get(timeout=120)
        assert not isinstance(res, str), res
        out[rank] = res
    for p in procs:
        p.join(timeout=30)
    for r in range(parties):
        assert out[r] == [parties] * rounds
