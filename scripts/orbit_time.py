"""Full-run wall time with orbit-compressed stages on / off (default run: sparse
prefix on; and every stage dense-or-compressed with the sparse prefix off).
Usage: python scripts/orbit_time.py [workload=c4]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
prob = shs.FactoringProblem.make(w["N"], w["a"])
eng = shs.IterativeShorEngine(prob, shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
print("orbit", eng.orbit_info(), "sparse stages", eng.sparse_stages(), flush=True)
for orbit in (True, False):
    eng.set_orbit(orbit)
    for sparse in (True, False):
        eng.set_sparse(sparse)
        eng.run(1, 0)
        ts, js = [], []
        for i in range(3):
            t0 = time.perf_counter()
            r = eng.run(1, 1 + i)
            ts.append(time.perf_counter() - t0)
            js.append(r.bits.j)
        print(f"orbit={orbit} sparse={sparse}: run {[round(x, 4) for x in ts]} s  j={js}", flush=True)
eng.close()
