"""The multi-process sharded path (one shard per torch.distributed rank, peers
attached through CUDA IPC handles: buffers, stage digits and ordering events)
with 2-3 ranks sharing the one GPU of this run. run() is the device-resident
loop (shs_shards_run): cross-rank order comes from IPC events, a shared-memory
host barrier only orders their enqueues, and no kernel waits on another rank's
kernel. run_stepwise() is the host-sequenced driver (gloo barrier/allreduce).
Both must equal the single-GPU engine (exact combine) bit for bit."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(1048351, 12345, 10, "force"), (4194301, 1234567, 8, "auto"), (262139, 31337, 9, "off")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2308_05047_b200 as shs
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        out = []
        for N, a, t, tiling in CASES:
            prob = shs.FactoringProblem.make(N, a, t)
            o = shs.SimulatorOptions(qubit_ceiling=64, combine="exact", tiling=tiling, device=0)
            shard = shs.Shard(prob, shs.ErrorConfig(), o, rank, world)
            eng = shs.ShardedShorEngine(prob, shs.ErrorConfig(), o, [shard],
                                        shs.DistGroup(shard, attach_ipc=True))
            for idx in range(2):
                r = eng.run(21, idx)  # device-resident: IPC events + shared-memory barrier
                w = eng.run_stepwise(21, idx)  # host-sequenced per-stage driver
                assert (w.bits.j, [x.p1 for x in w.trace]) == (r.bits.j, [x.p1 for x in r.trace])
                out.append((N, idx, r.bits.j, [x.p1 for x in r.trace]))
            dist.barrier()
            shard.close()
        q.put((rank, out))
    except Exception as exc:
        q.put((rank, f"{type(exc).__name__}: {exc}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_process_ipc_shards_match_single_engine(cuda_ok, world):
    import paper_2308_05047_b200 as shs
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, out = q.get(timeout=600)
        assert not isinstance(out, str), out
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
    for r in range(1, world):
        assert res[r] == res[0]
    k = 0
    for N, a, t, tiling in CASES:
        eng = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a, t), shs.ErrorConfig(),
                                      shs.SimulatorOptions(qubit_ceiling=64, combine="exact",
                                                           tiling=tiling))
        for idx in range(2):
            r = eng.run(21, idx)
            assert res[0][k] == (N, idx, r.bits.j, [x.p1 for x in r.trace]), (N, idx)
            k += 1
