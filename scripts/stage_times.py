"""Per-stage wall time of a full run through the step API (diagnostics)."""
import sys, time, json
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
N, a = int(sys.argv[1]), int(sys.argv[2])
tiling = sys.argv[3] if len(sys.argv) > 3 else "auto"
s0 = int(sys.argv[4]) if len(sys.argv) > 4 else 0
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64, tiling=tiling))
pows = eng.stage_multipliers()
eng.state_init()
prefix = 0
out = []
for s in range(s0, eng.t):
    eng.set_timing(True)
    t0 = time.perf_counter()
    p0, p1 = eng.stage_probs(s, prefix)
    t1 = time.perf_counter()
    b = shs.sample_measurement(p1, 1, 0, s, shs.ErrorConfig())["sampled_bit"]
    if s + 1 < eng.t:
        eng.stage_collapse(b, p1 if b else p0)
    t2 = time.perf_counter()
    kt = eng.kernel_times()
    pl = eng.tile_plan(s)
    out.append((s, pows[s], pl["tiled"], pl["H"], round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t1), 2),
                {k: round(v[0], 3) for k, v in kt.items()}))
    print(*out[-1], flush=True)
    prefix |= b << s
