import sys, time
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
for N, a in [(16777207, 2), (16777207, 3), (1048351, 12345), (268435247, 3)]:
    e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
    e.run(7, 0)
    t0 = time.perf_counter(); r = e.run(7, 1); dt = time.perf_counter() - t0
    nt = sum(e.tile_plan(s)["tiled"] for s in range(e.t))
    print(f"N={N} a={a}: {dt*1e3:.1f} ms/run {dt/e.t*1e3:.3f} ms/stage tiled {nt}/{e.t} j={r.bits.j}", flush=True)
