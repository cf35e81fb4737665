# A/B: lockstep probs with all loads batched, 80 regs (3 CTAs/SM, small spill) vs 120 regs (2 CTAs/SM)
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q -p no:cacheprovider > gpurun_out/pytest_lockab.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_lockab.log
for rep in 1 2; do
for lib in variants/lib_lb3.so variants/lib_lb2.so; do
  echo "=== $lib"
  SHS_LIB=$lib python scripts/lock_profile.py 262139 4242
  SHS_LIB=$lib python scripts/lock_profile.py 65521 5
  SHS_LIB=$lib python scripts/lock_profile.py 1048573 3
done; done
SHS_LIB=variants/lib_lb3.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lock_launches3.csv python scripts/lock_profile.py 262139 4242 > /dev/null 2>&1
SHS_LIB=variants/lib_lb2.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lock_launches3b.csv python scripts/lock_profile.py 262139 4242 > /dev/null 2>&1
