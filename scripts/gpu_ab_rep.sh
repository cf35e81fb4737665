#!/bin/bash
# ABAB repetitions of ab_stages.py over the given libs (config 4 and config 3)
for rep in 1 2 3; do
  for lib in "$@"; do
    echo "$rep $(basename $lib) c4 $(SHS_LIB=$lib timeout 300 python scripts/ab_stages.py 4294967213 5 50 6 2>&1 | tail -1)"
    echo "$rep $(basename $lib) c3 $(SHS_LIB=$lib timeout 300 python scripts/ab_stages.py 16777207 2 1 40 2>&1 | tail -1)"
  done
done
