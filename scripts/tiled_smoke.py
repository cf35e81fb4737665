"""Quick check of the tiled (TMA) path against the oracle at a small size."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2308_05047_b200 as shs
from oracle import Oracle, make_error
N, a, t = 262139, 31337, 6
o = Oracle()
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a, t), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64, tiling="force", combine="kahan"))
orc = o.engine(N, a, N.bit_length(), t, make_error())
print([eng.tile_plan(s)["tiled"] for s in range(t)], flush=True)
eng.state_init(); orc.state_init(); prefix = 0
for s in range(t):
    p = eng.stage_probs(s, prefix); q = orc.stage_probs(s, prefix, 0)
    d = np.ctypeslib.as_array(eng.stage_read(0, 0, N)); w = np.ctypeslib.as_array(orc.stage_read(0, 0, N))
    print(s, p == q, np.array_equal(d, w), flush=True)
    b = 1 if p[1] > 1e-300 and s % 2 else 0
    if p[b] < 1e-300: b = 1 - b
    if s + 1 < t:
        eng.stage_collapse(b, p[b]); orc.collapse(b, q[b])
    prefix |= b << s
