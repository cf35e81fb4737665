# Parity of the tiled paths after a kernel change, then mid-N timings.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_device_run.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_q.log
timeout 300 python scripts/c3_time.py > gpurun_out/c3_time.log 2>&1; echo "c3 rc $?"; cat gpurun_out/c3_time.log
timeout 300 python scripts/c3_breakdown.py > gpurun_out/c3_breakdown.log 2>&1; head -1 gpurun_out/c3_breakdown.log; sed -n 20,24p gpurun_out/c3_breakdown.log; tail -1 gpurun_out/c3_breakdown.log
