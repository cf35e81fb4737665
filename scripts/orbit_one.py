"""One default run (sparse prefix + orbit-compressed stages) of a workload, for ncu.
Usage: python scripts/orbit_one.py [workload=n30] [orbit=1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "n30"]
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(w["N"], w["a"]), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64))
eng.set_orbit(len(sys.argv) < 3 or sys.argv[2] != "0")
print(eng.orbit_info(), eng.run(1, 0).bits.j)
