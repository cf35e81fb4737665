#!/bin/bash
# config-4 last stages (small multipliers: direct / streams kernels) per lib
for lib in "$@"; do
  echo "== $(basename $lib)"
  SHS_LIB=$lib timeout 300 python scripts/stage_times.py 4294967213 5 auto 59 2>&1 | tail -4 | awk '{print $1, $2, $NF, $(NF-1), $(NF-2), $(NF-3), $(NF-4), $(NF-5)}'
done
