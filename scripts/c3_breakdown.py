"""Per-stage kernel times (CUDA events on the engine stream) of a config-3 run
through the step API: which stages / passes keep mid-N below the roofline."""
import sys
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs

N, a = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (16777207, 2)
e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(),
                            shs.SimulatorOptions(qubit_ceiling=64))
e.run(7, 0)
e.set_timing(True)
e.run(7, 1)
kt = e.kernel_times()
print("run totals (ms, launches):", {k: (round(v[0], 3), v[1]) for k, v in kt.items()})
e.set_timing(False)
e.set_timing(True)
e.state_init()
prev = {k: 0.0 for k in kt}
rows = []
prefix = 0
for s in range(e.t):
    p0, p1 = e.stage_probs(s, prefix)
    b = 1 if p1 > p0 else 0
    if s + 1 < e.t:
        e.stage_collapse(b, p1 if b else p0)
    prefix |= b << s
    kt = e.kernel_times()
    d = {k: kt[k][0] - prev[k] for k in kt}
    prev = {k: kt[k][0] for k in kt}
    pl = e.tile_plan(s)
    A = e.stage_multipliers()[s]
    rows.append((s, A, pl["tiled"], pl["H"], d["probs"], d["combine"], d["collapse"]))
bpa = N * 16
tot = 0
for s, A, tl, H, pr, cb, co in rows:
    tot += pr + cb + co
    print(f"s={s:2d} A={A:>9d} tiled={tl} H={H:6d} probs {pr*1e3:7.1f} us ({2*bpa/pr/1e6 if pr else 0:6.0f} GB/s)"
          f" fin {cb*1e3:5.1f} us collapse {co*1e3:7.1f} us ({3*bpa/co/1e6 if co else 0:6.0f} GB/s)")
print(f"sum of kernel time {tot:.3f} ms = {tot/e.t*1e3:.1f} us/stage; roofline {80*N/6548.5e9*1e6:.1f} us/stage")
