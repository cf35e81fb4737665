#!/bin/bash
# per-kernel durations (ncu launch list) of config-4 tiled stages 57-59, per lib
for lib in "$@"; do
  n=$(basename $lib .so)
  SHS_LIB=$lib timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tiled --csv --log-file gpurun_out/abn_$n.csv python scripts/stage_times.py 4294967213 5 auto 57 > /dev/null 2>&1
  echo "$n rc $?"
done
