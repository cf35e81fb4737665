"""Batched small-N throughput + a correctness spot check against the per-stage path."""
import sys, time, math
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
for N, a, count in [(15, 7, 200000), (21, 2, 100000), (35, 4, 100000), (4087, 1001, 20000), (1001, 10, 20000)]:
    e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a, min(shs.recommended_t(N), 20)), shs.ErrorConfig(),
                                shs.SimulatorOptions(qubit_ceiling=64))
    import numpy as np
    buf = np.empty((count, 2), dtype=np.uint64)
    e.run_batch_array(2, 0, count, buf)
    t0 = time.perf_counter(); e.run_batch_array(2, 0, count, buf); dt = time.perf_counter() - t0
    ok = [int(x) for x in buf[:50, 0]] == e.run_sequential(2, 0, 50)
    print(f"N={N} t={e.t}: {count/dt/1e6:.2f} M runs/s ({dt*1e3:.1f} ms for {count}) match={ok}", flush=True)
