#!/bin/bash
# config-3 full-run time per lib (A/B of tile-plan parameters), 2 repetitions
for rep in 1 2; do for lib in "$@"; do
  echo "$rep $(basename $lib) $(SHS_LIB=$lib timeout 300 python scripts/c3_time.py 2>&1 | head -2 | tr '\n' ' ')"
done; done
