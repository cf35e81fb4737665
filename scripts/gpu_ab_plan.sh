#!/bin/bash
# A/B of tile-plan parameters: config-3 run time and config-4 tiled stages per variant lib
for lib in paper_2308_05047_b200/libshorsim_b200.so build/lib_*.so; do
  echo "== $lib"
  SHS_LIB=$lib timeout 300 python scripts/c3_time.py 2>&1 | head -2
  SHS_LIB=$lib timeout 300 python scripts/stage_times.py 4294967213 5 auto 56 2>&1 | head -4 | awk '{print $1,$2,$3,$4,$5,$6}'
done
