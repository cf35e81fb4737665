for b in default 8 16 32 64 256; do
  if [ $b = default ]; then unset SHS_LOCK_BATCH; else export SHS_LOCK_BATCH=$b; fi
  echo "=== SHS_LOCK_BATCH=$b"; python scripts/create_cost.py
done
