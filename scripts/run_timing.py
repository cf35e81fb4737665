"""Wall time vs summed kernel times (CUDA events per launch group) of a default
run() (sparse prefix) and a dense one at config 4."""
import sys, time
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
N, a = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (4294967213, 5)
e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
for sp in (True, False):
    e.set_sparse(sp)
    e.run(7, 0)
    e.set_timing(True)
    t0 = time.perf_counter(); e.run(7, 1); wall = time.perf_counter() - t0
    kt = e.kernel_times()
    e.set_timing(False)
    tot = sum(v[0] for v in kt.values())
    print(f"sparse={sp} stages={e.sparse_stages()} wall {wall*1e3:.1f} ms, kernels {tot:.1f} ms", {k: (round(v[0], 1), v[1]) for k, v in kt.items()})
    t0 = time.perf_counter(); e.run(7, 2); print(f"  untimed wall {1e3*(time.perf_counter()-t0):.1f} ms")
