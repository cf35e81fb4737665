# A/B of ring depth / norm buffers (probs smem budget) at config 4, alternating with the tree
for rep in 1 2; do
for lib in paper_2308_05047_b200/libshorsim_b200.so variants/lib_r3n6.so variants/lib_r5n2.so variants/lib_r4n3.so; do
  echo "=== $lib"
  SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-small --steps 12 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json | cut -c1-170
done
done
