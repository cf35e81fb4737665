# A/B: evict-first collapse stores (tree) vs plain (variants/lib_nocs.so)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "tiled or forced" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_q.log
for rep in 1 2; do
for lib in variants/lib_nocs.so paper_2308_05047_b200/libshorsim_b200.so; do
  echo "=== $lib"
  SHS_LIB=$lib timeout 300 python scripts/c3_time.py 2>&1 | head -1
  SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-small --steps 12 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json | cut -c1-200
done
done
CMD="python bench.py --workload n30 --steps 3 --warmup 3 --no-cpu-baseline --no-small"
for lib in variants/lib_nocs.so paper_2308_05047_b200/libshorsim_b200.so; do
SHS_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_tiled<0" -c 2 $CMD 2>/dev/null | grep -E "k_tiled|duration|bytes" | head -8
done
