# lockstep buffers kept across calls: parity + wall time (3 reps each)
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_dropin.py -x -q -p no:cacheprovider > gpurun_out/pytest_lockkeep.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_lockkeep.log
for rep in 1 2 3; do python scripts/lock_profile.py 262139 4242; python scripts/lock_profile.py 65521 5; done
python scripts/lock_profile.py 1048573 3; python scripts/create_cost.py
