timeout 120 python scripts/tiled_smoke.py > gpurun_out/tiled_smoke.log 2>&1; rc=$?; echo "tiled smoke rc $rc"; if [ $rc -ne 0 ]; then tail -3 gpurun_out/tiled_smoke.log; exit 1; fi
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_random.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_q.log
timeout 900 python bench.py --no-cpu-baseline --no-small > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc $?"; python scripts/summarize_bench.py gpurun_out/bench_c4.json
python -c "import json;d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]);print(json.dumps(d.get('config3_error_models'),indent=0))"
