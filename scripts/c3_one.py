"""One config-3 run (N = 16777207, a = 2) with every stage swept, for ncu captures
(profiles/r02/ncu_c3_orbit_tiled.json). Usage: python scripts/c3_one.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402

eng = shs.IterativeShorEngine(shs.FactoringProblem.make(16777207, 2), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64))
eng.set_sparse(False)
eng.run(1, 0)
print(eng.run(1, 1).bits.j)
