timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_device_run.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_q.log
for v in 0 1; do
  echo "=== SHS_STREAM_PROBS=$v"
  SHS_STREAM_PROBS=$v timeout 300 python scripts/c3_breakdown.py 4294967213 5 > gpurun_out/c4_sp_$v.log 2>&1; grep -E "^s=6[123] " gpurun_out/c4_sp_$v.log | cut -c1-150
  SHS_STREAM_PROBS=$v python scripts/run_timing.py 2>&1 | head -1
  SHS_STREAM_PROBS=$v timeout 300 python scripts/c3_breakdown.py 16777207 2 > gpurun_out/c3_sp_$v.log 2>&1; grep -E "^s=4[4567] " gpurun_out/c3_sp_$v.log | cut -c1-150
done
