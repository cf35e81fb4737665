import sys
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
e = shs.IterativeShorEngine(shs.FactoringProblem.make(15, 7, 8), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
e.run_batch(2, 0, 1000)
e.run_batch(2, 0, 200000)
print("ok")
