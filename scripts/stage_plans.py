"""Per stage: tile plan, whether it runs orbit-compressed. Usage: python scripts/stage_plans.py [workload=c4]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(w["N"], w["a"]), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64))
orb = eng.orbit_stages()
mult = eng.stage_multipliers()
for s in range(eng.problem.t):
    print(s, mult[s], eng.tile_plan(s), "orbit" if orb[s] else "")
