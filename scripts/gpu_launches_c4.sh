# ncu launch list (durations only, cold, serialised) of the default config-4 bench command
timeout 1300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/v16_launches_c4.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-small > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc $?"
