for lib in paper_2308_05047_b200/libshorsim_b200.so build/lib_avg640.so build/lib_min1.so build/lib_both1.so build/lib_both2.so; do
  echo "=== $lib"
  SHS_LIB=$lib timeout 300 python scripts/c3_time.py
  SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-small --steps 10 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json
done
