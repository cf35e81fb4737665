"""Host cost of one campaign problem: engine creation, 256 shots (lockstep), close
(median / max over 20 problems of each size)."""
import math
import statistics
import sys
import time
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs

for N, a in [(4087, 1001), (65521 * 3 + 2, 5), (262139, 4242)]:
    if math.gcd(a, N) != 1:
        a += 1
    p = shs.FactoringProblem.make(N, a)
    o = shs.SimulatorOptions(qubit_ceiling=64)
    shs.IterativeShorEngine(p, shs.ErrorConfig(), o).close()
    tc, tr, tx = [], [], []
    for i in range(20):
        t0 = time.perf_counter(); e = shs.IterativeShorEngine(p, shs.ErrorConfig(), o); t1 = time.perf_counter()
        e.run_batch_array(1, 0, 256); t2 = time.perf_counter()
        e.close(); t3 = time.perf_counter()
        tc.append(t1 - t0); tr.append(t2 - t1); tx.append(t3 - t2)
    f = lambda v: f"{1e3 * statistics.median(v):.2f} (max {1e3 * max(v):.2f}) ms"
    print(f"N={N} t={p.t}: create {f(tc)}, 256 shots {f(tr)}, close {f(tx)}", flush=True)
