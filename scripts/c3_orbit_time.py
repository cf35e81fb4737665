import sys, time
sys.path.insert(0, '.')
import paper_2308_05047_b200 as shs
for N, a in [(16777207, 2), (16777207, 1234567)]:
    eng = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
    print(N, a, eng.orbit_info(), "sparse", eng.sparse_stages())
    for orbit in (True, False):
        eng.set_orbit(orbit)
        js = []
        eng.run(1, 0)
        t0 = time.perf_counter()
        for i in range(20):
            js.append(eng.run(1, i + 1).bits.j)
        print(f"  orbit={orbit}: {1e3*(time.perf_counter()-t0)/20:.2f} ms per run", hash(tuple(js)) % 100000)
    eng.close()
