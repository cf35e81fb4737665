timeout 900 python -m pytest tests/test_gpu_device_run.py -x -q -p no:cacheprovider > gpurun_out/pytest_sp.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_sp.log
python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_2308_05047_b200 as shs
for N, a in [(16777207, 2), (268435247, 3), (4294967213, 5)]:
    e = shs.IterativeShorEngine(shs.FactoringProblem.make(N, a), shs.ErrorConfig(), shs.SimulatorOptions(qubit_ceiling=64))
    for sp in (False, True):
        e.set_sparse(sp)
        e.run(7, 0)
        t0 = time.perf_counter(); r = e.run(7, 1); dt = time.perf_counter() - t0
        print(f"N={N} a={a} sparse={e.sparse_stages()}: {dt*1e3:.1f} ms/run j={r.bits.j}", flush=True)
    e.close()
PY
