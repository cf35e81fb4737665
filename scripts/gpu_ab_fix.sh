# A/B of k_tile_fixup versions: variants/lib_head.so (CTA-staged, 1 folding warp) vs the tree (all warps fold).
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -x -q -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_q.log
for rep in 1 2; do
for lib in variants/lib_head.so paper_2308_05047_b200/libshorsim_b200.so; do
  echo "=== $lib"
  SHS_LIB=$lib timeout 300 python scripts/c3_time.py 2>&1 | head -2
  SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-small --steps 12 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json | cut -c1-200
done
done
SHS_LIB=paper_2308_05047_b200/libshorsim_b200.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tile_fixup" -c 8 --csv python scripts/c3_one_run.py 2>/dev/null | grep -v "^==" | tail -8 | cut -d, -f5,15,16
