timeout 900 python -m pytest tests/test_gpu_batch.py -x -q -p no:cacheprovider > gpurun_out/pytest_lock.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_lock.log
python - <<'PY'
import sys, time, os
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
for N, a, M in [(4087, 1001, 1024), (65521, 3, 1024), (262139, 4242, 256)]:
    e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
    e.run_batch_array(1, 0, 8)
    t0 = time.perf_counter(); e.run_batch_array(1, 0, M); dt = time.perf_counter() - t0
    t1 = time.perf_counter(); [e.run(1, i) for i in range(32)]; ds = (time.perf_counter() - t1) / 32
    print(f"N={N} t={e.t}: lockstep {M / dt:.0f} runs/s; single run() {1 / ds:.0f} runs/s", flush=True)
    e.close()
PY
