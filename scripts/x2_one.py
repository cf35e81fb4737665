"""One device-resident sharded run (v2 exchange) for profiling: python scripts/x2_one.py n30 8"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "n30"]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
prob = shs.FactoringProblem.make(w["N"], w["a"])
eng = shs.ShardedShorEngine.virtual(prob, shs.ErrorConfig(),
                                    shs.SimulatorOptions(qubit_ceiling=64, combine="exact"), nshards=G)
eng.run(1, 0)
eng.run(1, 1)
print("ok")
