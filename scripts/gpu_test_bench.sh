# GPU round trip: parity tests, then the c4 bench and the n29 profiling-size bench.
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -25 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc $?"
timeout 600 python bench.py --workload n29 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n29.json 2> gpurun_out/bench_n29.err; echo "bench n29 rc $?"
python - <<'PY'
import json
for f in ["gpurun_out/bench_c4.json", "gpurun_out/bench_n29.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "ms/stage %.2f" % d["ms_per_step"], "stage frac %.3f" % d["stage_frac_of_hbm"],
              {k: (round(v["avg_ms"], 3), v["achieved_gbs"] and round(v["achieved_gbs"])) for k, v in d["kernels"].items()},
              "s/run %.2f" % d["s_per_run"], d["clocks"])
    except Exception as e:
        print(f, "ERR", e)
PY
tail -5 gpurun_out/bench_c4.err
