"""Exchange v1 vs v2 on ONE GPU with G virtual shards (in-process): per-kernel
CUDA-event times of one timed device-resident run, and the HBM bytes each
exchange moves per stage (on one GPU the "link" is local HBM).
Usage: python scripts/x2_probe.py [workload=n29] [G=2]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS, peaks  # noqa: E402


def probe(workload, G, v1):
    if v1:
        os.environ["SHS_EXCHANGE"] = "1"
    else:
        os.environ.pop("SHS_EXCHANGE", None)
    w = WORKLOADS[workload]
    prob = shs.FactoringProblem.make(w["N"], w["a"])
    opts = shs.SimulatorOptions(qubit_ceiling=64, combine="exact")
    eng = shs.ShardedShorEngine.virtual(prob, shs.ErrorConfig(), opts, nshards=G)
    eng.run(1, 0)  # prepare + warm
    import time
    t0 = time.perf_counter()
    r = eng.run(1, 1)
    run_s = time.perf_counter() - t0
    for sh in eng.shards:
        sh.set_timing(True)
    eng.run(1, 2)
    out = {"workload": workload, "G": G, "exchange": "v1" if v1 else "v2", "N": w["N"],
           "t": prob.t, "run_s": run_s, "j": str(r.bits.j)}
    S = eng.shards[0].hi - eng.shards[0].lo
    tot = {}
    for sh in eng.shards:
        for k, (ms, n) in sh.kernel_times().items():
            a = tot.setdefault(k, [0.0, 0])
            a[0] += ms
            a[1] += n
    out["kernel_avg_ms"] = {k: v[0] / v[1] for k, v in tot.items() if v[1]}
    out["launches"] = {k: v[1] for k, v in tot.items()}
    hbm, _ = peaks()
    if not v1 and tot.get("pack", [0, 0])[1]:
        # pack per launch: reads its S/K sources, writes S/K elements (16 B each)
        K = eng.shards[0]._lib.shs_shard_launch_count  # (not used)
        K = max(1, round(tot["pack"][1] / max(1, tot["probs"][1] - G)))
        out["rounds"] = K
        per = 32 * S / K
        out["pack_gbs"] = per / (out["kernel_avg_ms"]["pack"] * 1e-3) / 1e9
        out["unpack_gbs"] = per / (out["kernel_avg_ms"]["unpack"] * 1e-3) / 1e9
    if v1 and tot["exchange"][1]:
        # v1 executor: every element read once and written once (32 B) per stage over all ranks
        out["exchange_gbs_per_shard_launch"] = 32 * S / (out["kernel_avg_ms"]["exchange"] * 1e-3) / 1e9
    out["hbm_peak"] = hbm
    eng.close()
    return out


if __name__ == "__main__":
    wl = sys.argv[1] if len(sys.argv) > 1 else "n29"
    G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    for v1 in (False, True):
        print(json.dumps(probe(wl, G, v1)))
