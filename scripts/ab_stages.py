"""Mean device time of the tiled probs / collapse kernels over config-4 stages
s0+1 .. s0+n (diagnostics for A/B of kernel variants; SHS_LIB picks the lib)."""
import sys
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
N, a = int(sys.argv[1]), int(sys.argv[2])
s0, n = int(sys.argv[3]), int(sys.argv[4])
eng = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(),
                              shs.SimulatorOptions(qubit_ceiling=64))
eng.state_init()
prefix, tp, tc, k = 0, 0.0, 0.0, 0
for s in range(s0, min(s0 + n + 1, eng.t - 1)):
    eng.set_timing(True)
    p0, p1 = eng.stage_probs(s, prefix)
    b = 1 if p1 >= p0 else 0
    eng.stage_collapse(b, p1 if b else p0)
    kt = eng.kernel_times()
    if s > s0:
        tp += kt["probs"][0]; tc += kt["collapse"][0]; k += 1
    prefix |= b << s
print(f"probs {tp / k:.3f} collapse {tc / k:.3f} ms over {k} stages")
