# A/B of tiled-kernel shapes: parity subset + config-4 and n29 benches per build variant
for lib in paper_2308_05047_b200/libshorsim_b200.so build/lib_r16c64s5.so build/lib_r32c32.so build/lib_r32c32s5.so build/lib_r16c32s8.so; do
  echo "=== $lib"
  SHS_LIB=$lib timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "forced_sequence_vs_oracle and force" > gpurun_out/ab_pytest.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/ab_pytest.log
  SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json
  SHS_LIB=$lib timeout 300 python bench.py --workload n29 --no-cpu-baseline --steps 10 > gpurun_out/ab_n29.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_n29.json
done
