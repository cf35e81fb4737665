import sys, math, random
sys.path.insert(0, '/root/repo')
import paper_2308_05047_b200 as shs
rng = random.Random(1)
bad = 0
for trial in range(400):
    L = rng.randrange(13, 19)
    N = rng.randrange(1 << (L - 1), 1 << L) | 1
    a = rng.randrange(2, N - 1)
    if math.gcd(a, N) != 1: continue
    prob = shs.FactoringProblem.make(N, a)
    eng = shs.IterativeShorEngine(prob, shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
    try:
        eng.run_many(3, 0, 1)
        eng.run_many(3, 1, 7)
    except Exception as exc:
        bad += 1
        print("FAIL", N, a, prob.t, eng._lib.shs_num_blocks(eng._h), type(exc).__name__, exc)
        if bad > 5: break
    eng.close()
print("done bad", bad)
