timeout 120 python scripts/tiled_smoke.py > gpurun_out/tiled_smoke.log 2>&1; rc=$?; echo "tiled smoke rc $rc"; cat gpurun_out/tiled_smoke.log | tail -8
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -8 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc $?"
python scripts/summarize_bench.py gpurun_out/bench_c4.json
timeout 600 python bench.py --workload n29 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n29.json 2> gpurun_out/bench_n29.err; echo "n29 rc $?"
python scripts/summarize_bench.py gpurun_out/bench_n29.json
