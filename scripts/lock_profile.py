"""One campaign-size problem through the lockstep multi-shot path (run_problem's
256 shots), for an ncu launch list: python scripts/lock_profile.py [N] [a]."""
import sys, time
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 262139
a = int(sys.argv[2]) if len(sys.argv) > 2 else 4242
p = shs.FactoringProblem.make(N, a)
o = shs.SimulatorOptions(qubit_ceiling=64)
with shs.IterativeShorEngine(p, shs.ErrorConfig(), o) as e:
    e.run_batch_array(1, 0, 256)  # warm-up
    t0 = time.perf_counter()
    e.run_batch_array(1, 0, 256)
    t1 = time.perf_counter()
    for i in range(8):
        e.run(1, i)
    t2 = time.perf_counter()
print(f"N={N} t={p.t}: 256 shots {1e3 * (t1 - t0):.2f} ms, single run {1e3 * (t2 - t1) / 8:.3f} ms",
      flush=True)
