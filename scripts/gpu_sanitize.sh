timeout 900 python -m pytest tests/test_gpu_random.py -x -q -p no:cacheprovider > gpurun_out/pytest_random.log 2>&1; echo "random rc $?"; tail -3 gpurun_out/pytest_random.log
# memcheck on the tiled (single-GPU) and sharded small cases; only after both ran clean above
timeout 120 python scripts/tiled_smoke.py > /dev/null 2>&1 && timeout 120 python scripts/shard_smoke.py > /dev/null 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/tiled_smoke.py > gpurun_out/memcheck_tiled.log 2>&1; echo "memcheck tiled rc $?"; tail -4 gpurun_out/memcheck_tiled.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/shard_smoke.py > gpurun_out/memcheck_shard.log 2>&1; echo "memcheck shard rc $?"; tail -4 gpurun_out/memcheck_shard.log
