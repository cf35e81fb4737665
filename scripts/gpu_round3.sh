timeout 120 python scripts/shard_smoke.py > gpurun_out/shard_smoke.log 2>&1; rc=$?; echo "shard smoke rc $rc"; tail -5 gpurun_out/shard_smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc $?"
python scripts/summarize_bench.py gpurun_out/bench_c4.json
