"""Timeline of one device-resident sharded run (G virtual shards on one GPU,
exchange v2 in K rounds): every launch's start / end on its own stream
(shs_shard_timeline), and how much of the pack kernels' time runs concurrently
with an unpack (the exchange of round g+1 overlapping the on-shard scatter of
round g). Usage: SHS_X2_ROUNDS=3 python scripts/x2_timeline.py n31 2 [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "n31"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = WORKLOADS[wl]
prob = shs.FactoringProblem.make(w["N"], w["a"])
eng = shs.ShardedShorEngine.virtual(prob, shs.ErrorConfig(),
                                    shs.SimulatorOptions(qubit_ceiling=64, combine="exact"),
                                    nshards=G)
eng.run(1, 0)  # prepare + warm
for sh in eng.shards:
    sh.set_timeline(True)
eng.run(1, 1)
tl = {q: sh.timeline() for q, sh in enumerate(eng.shards)}


def overlap(a, b):
    return max(0.0, min(a[2], b[2]) - max(a[1], b[1]))


out = {"workload": wl, "G": G, "rounds": os.environ.get("SHS_X2_ROUNDS", "auto"), "shards": {}}
for q, ev in tl.items():
    packs = [e for e in ev if e[0] == "pack"]
    unpacks = [e for e in ev if e[0] == "unpack"]
    locs = [e for e in ev if e[0] in ("probs", "collapse")]
    pack_t = sum(e[2] - e[1] for e in packs)
    ov = sum(overlap(p, u) for p in packs for u in unpacks)  # same shard
    ov_any = sum(overlap(p, u) for p in packs for qq in tl for u in tl[qq] if u[0] == "unpack")
    span = max(e[2] for e in ev) - min(e[1] for e in ev)
    out["shards"][q] = {"launches": len(ev), "pack_ms": pack_t,
                        "unpack_ms": sum(e[2] - e[1] for e in unpacks),
                        "local_ms": sum(e[2] - e[1] for e in locs),
                        "pack_overlapping_own_unpack_ms": ov,
                        "pack_overlapping_any_unpack_ms": ov_any, "run_span_ms": span}
    if q == 0:  # one stage of shard 0 in detail: the first stage with a pack
        first = next(i for i, e in enumerate(ev) if e[0] == "pack")
        out["shard0_first_exchange_stage"] = [(k, round(a, 3), round(b, 3))
                                              for k, a, b in ev[first:first + 12]]
print(json.dumps(out, indent=1))
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as f:
        json.dump({"summary": out, "timeline": tl}, f)
