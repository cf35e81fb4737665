# Device-resident run: parity vs the host-driven loop, then c3/c4 timings A/B.
timeout 900 python -m pytest tests/test_gpu_device_run.py -x -q -p no:cacheprovider > gpurun_out/pytest_dev.log 2>&1; echo "pytest dev rc $?"; tail -15 gpurun_out/pytest_dev.log
timeout 300 python scripts/c3_time.py > gpurun_out/c3_dev.log 2>&1; echo "c3 dev rc $?"; cat gpurun_out/c3_dev.log
SHS_HOST_MEASURE=1 timeout 300 python scripts/c3_time.py > gpurun_out/c3_host.log 2>&1; echo "c3 host rc $?"; cat gpurun_out/c3_host.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-small > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc $?"; python scripts/summarize_bench.py gpurun_out/bench_c4.json
python -c "import json;d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]);print(json.dumps(d.get('config3_error_models')))"
