timeout 900 python -m pytest tests/test_gpu_postprocess.py -x -q -p no:cacheprovider > gpurun_out/pytest_pp.log 2>&1; echo "pytest pp rc $?"; tail -15 gpurun_out/pytest_pp.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_pp.json 2> gpurun_out/bench_pp.err; echo "bench rc $?"; tail -3 gpurun_out/bench_pp.err
python -c "import json;d=json.loads(open('gpurun_out/bench_pp.json').read().strip().splitlines()[-1]);print(json.dumps(d.get('batched_small_n'),indent=1))"
