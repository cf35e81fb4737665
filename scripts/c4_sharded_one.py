"""One full config-4 run through the multi-device engine (2 virtual shards of one GPU), for ncu launch lists."""
import sys

sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs  # noqa: E402

prob = shs.FactoringProblem.make(4294967213, 5)
eng = shs.IterativeShorEngine(prob, shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64,
                                                                            devices=[0, 0]))
eng.run(1, 0)
print(eng.run(1, 1).bits.j)
