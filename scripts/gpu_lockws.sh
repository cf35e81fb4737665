# A/B: warp-specialized lockstep probs (default) vs k_lock_probs (SHS_LOCK_WS=0)
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_dropin.py -x -q -p no:cacheprovider > gpurun_out/pytest_lockws.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_lockws.log
for rep in 1 2; do for ws in 1 0; do echo "=== SHS_LOCK_WS=$ws"
SHS_LOCK_WS=$ws python scripts/lock_profile.py 262139 4242; SHS_LOCK_WS=$ws python scripts/lock_profile.py 65521 5; SHS_LOCK_WS=$ws python scripts/lock_profile.py 1048573 3
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lock_launches_ws.csv python scripts/lock_profile.py 262139 4242 > /dev/null 2>&1; echo "ncu rc $?"
