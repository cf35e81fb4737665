"""Wall time of full config-4 runs through the multi-device engine with 2 virtual
shards of one GPU (devices=[0, 0]: sparse prefix, exchange v2 in K rounds)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs  # noqa: E402

prob = shs.FactoringProblem.make(4294967213, 5)
eng = shs.IterativeShorEngine(prob, shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64,
                                                                            devices=[0, 0]))
eng.run(1, 0)
ts = []
for i in range(3):
    t0 = time.perf_counter()
    r = eng.run(1, 1 + i)
    ts.append(time.perf_counter() - t0)
eng.set_sparse(False)
t0 = time.perf_counter()
eng.run(1, 9)
dense = time.perf_counter() - t0
print("c4 sharded (2 virtual shards): run", [round(x, 3) for x in ts], "s; every stage dense",
      round(dense, 3), "s")
