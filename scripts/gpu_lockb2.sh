nproc; uptime
for rep in 1 2; do
for b in default 256; do
  if [ $b = default ]; then unset SHS_LOCK_BATCH; else export SHS_LOCK_BATCH=$b; fi
  echo "=== SHS_LOCK_BATCH=$b"; python scripts/create_cost.py | tail -2
done; done
