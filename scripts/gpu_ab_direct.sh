# A/B of the direct (small-multiplier / first-stage) kernels at config 4: v8 library vs the tree.
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_device_run.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_q.log
for lib in variants/lib_v8.so paper_2308_05047_b200/libshorsim_b200.so; do
  SHS_LIB=$lib timeout 300 python scripts/c3_breakdown.py 4294967213 5 > gpurun_out/c4_bd_$(basename $lib).log 2>&1
  echo "== $lib"; head -3 gpurun_out/c4_bd_$(basename $lib).log | cut -c1-150; tail -4 gpurun_out/c4_bd_$(basename $lib).log
done
timeout 300 python scripts/c3_time.py > gpurun_out/c3_time.log 2>&1; cat gpurun_out/c3_time.log
