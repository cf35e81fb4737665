# lockstep speculative group-0 write: parity, then A/B vs the previous library (variants/lib_head.so) and SHS_SPEC=0
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_dropin.py -x -q -p no:cacheprovider > gpurun_out/pytest_lockspec.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_lockspec.log
for rep in 1 2; do for v in head spec off; do echo "=== $v"
lib=paper_2308_05047_b200/libshorsim_b200.so; [ $v = head ] && lib=variants/lib_head.so; sp=1; [ $v = off ] && sp=0
SHS_LIB=$lib SHS_SPEC=$sp python scripts/lock_profile.py 262139 4242; SHS_LIB=$lib SHS_SPEC=$sp python scripts/lock_profile.py 65521 5; SHS_LIB=$lib SHS_SPEC=$sp python scripts/lock_profile.py 1048573 3
done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v15_launches_lock.csv python scripts/lock_profile.py 262139 4242 > /dev/null 2>&1; echo "ncu lock rc $?"
CMD="python bench.py --workload n30 --steps 3 --warmup 3 --no-cpu-baseline --no-small"
timeout 300 $CMD > gpurun_out/v15_bench_n30.json 2>&1; echo "n30 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tiled" -s 2 -c 2 -o gpurun_out/v15_prof_n30 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"; tail -2 gpurun_out/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v15_launches_n30.csv $CMD > /dev/null 2>&1; echo "ncu n30 list rc $?"
