for d in 64 32 16 8; do
SHS_SPARSE_DENSITY=$d python - <<'PY'
import sys, time, os
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
for N, a in [(16777207, 2), (4294967213, 5)]:
    e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
    e.run(7, 0)
    best = 1e9
    for i in range(3 if N < 1e9 else 2):
        t0 = time.perf_counter(); r = e.run(7, 1); best = min(best, time.perf_counter() - t0)
    print(f"density {os.environ['SHS_SPARSE_DENSITY']} N={N} sparse={e.sparse_stages()}: {best*1e3:.1f} ms/run j={r.bits.j}", flush=True)
    e.close()
PY
done
