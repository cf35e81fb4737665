import sys
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
e = shs.IterativeShorEngine(shs.FactoringProblem.make(16777207, 2), shs.ErrorConfig(),
                            shs.SimulatorOptions(qubit_ceiling=64))
for i in range(2):
    e.run(7, i)
print("ok")
