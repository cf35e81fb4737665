# A/B at config 4: the split work variant for plans with < 16 bands per SM (default) vs round-robin for all (SHS_TILE_SPLIT=0)
for rep in 1 2; do
for v in default 0; do
  if [ $v = default ]; then unset SHS_TILE_SPLIT; else export SHS_TILE_SPLIT=0; fi
  echo "=== SHS_TILE_SPLIT=$v"
  timeout 300 python scripts/c3_breakdown.py 4294967213 5 > gpurun_out/c4_bd_$v.log 2>&1; grep -E "^s=(16|20|22) " gpurun_out/c4_bd_$v.log | cut -c1-140; tail -1 gpurun_out/c4_bd_$v.log
done
done
unset SHS_TILE_SPLIT
