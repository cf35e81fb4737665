"""Device time of one stage's probs pass (CUDA events on the engine stream), orbit
on / off, through the step API with norm checks off (also usable with the
SHS_ORB_EXP timing-experiment builds, whose numbers are not results).
Usage: python scripts/orbit_kernel_time.py [workload=n30] [stage=40] [orbit=1]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2308_05047_b200 as shs  # noqa: E402
from bench import WORKLOADS  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "n30"]
s = int(sys.argv[2]) if len(sys.argv) > 2 else 40
orbit = len(sys.argv) < 4 or sys.argv[3] != "0"
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(w["N"], w["a"]), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64, check_norms=False))
eng.set_orbit(orbit)
eng.state_init()
p0, p1 = eng.stage_probs(0, 0)
eng.stage_collapse(0, p0)
eng.stage_probs(s, 0)  # (dense -> compressed on the first orbit stage)
eng.set_timing(True)
for _ in range(5):
    eng.stage_probs(s, 0)
kt = eng.kernel_times()
print(f"orbit={orbit} stage {s}: probs pass {kt['probs'][0] / kt['probs'][1]:.3f} ms", flush=True)
