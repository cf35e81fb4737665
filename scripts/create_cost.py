"""Host cost of one campaign problem: engine creation, 256 shots (lockstep), close."""
import sys, time
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
for N, a in [(4087, 1001), (65521 * 3 + 2, 5), (262139, 4242)]:
    import math
    if math.gcd(a, N) != 1:
        a += 1
    p = shs.FactoringProblem.make(N, a)
    o = shs.SimulatorOptions(qubit_ceiling=64)
    shs.IterativeShorEngine(p, shs.ErrorConfig(), o).close()
    tc = tr = tx = 0.0
    n = 20
    for i in range(n):
        t0 = time.perf_counter(); e = shs.IterativeShorEngine(p, shs.ErrorConfig(), o); t1 = time.perf_counter()
        e.run_batch_array(1, 0, 256); t2 = time.perf_counter()
        e.close(); t3 = time.perf_counter()
        tc += t1 - t0; tr += t2 - t1; tx += t3 - t2
    print(f"N={N} t={p.t}: create {1e3*tc/n:.2f} ms, 256 shots {1e3*tr/n:.2f} ms, close {1e3*tx/n:.2f} ms", flush=True)
