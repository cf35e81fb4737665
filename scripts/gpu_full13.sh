python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/v13_bench_c4.json 2> gpurun_out/v13_bench_c4.err; echo "bench rc $?"; tail -2 gpurun_out/v13_bench_c4.err
python scripts/summarize_bench.py gpurun_out/v13_bench_c4.json | cut -c1-500
python -c "import json;d=json.loads(open('gpurun_out/v13_bench_c4.json').read().strip().splitlines()[-1]);print(json.dumps(d['batched_small_n']['config2_N21_N35'].get('statistics')))"
python -c "import json;d=json.loads(open('gpurun_out/v13_bench_c4.json').read().strip().splitlines()[-1]);print(json.dumps(d['batched_small_n']['campaign_L18_lockstep']))"
python scripts/lock_profile.py 262139 4242; python scripts/lock_profile.py 65521 5; python scripts/lock_profile.py 1048573 3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v13_launches_lock.csv python scripts/lock_profile.py 262139 4242 > /dev/null 2>&1; echo "ncu rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v13_launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c4 rc $?"
timeout 300 python bench.py --impl reference > gpurun_out/v13_bench_reference.json 2>/dev/null; echo "ref rc $?"
