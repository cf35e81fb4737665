for lib in paper_2308_05047_b200/libshorsim_b200.so build/lib_r64c16.so build/lib_r64c16nb2.so; do
  echo "=== $lib"
  SHS_LIB=$lib timeout 120 python scripts/tiled_smoke.py > gpurun_out/ab_smoke.log 2>&1; rc=$?; echo "smoke rc $rc"; if [ $rc -ne 0 ]; then tail -3 gpurun_out/ab_smoke.log; continue; fi
  SHS_LIB=$lib timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider -k "force or tile or virtual" > gpurun_out/ab_pytest.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/ab_pytest.log
  SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json
  SHS_LIB=$lib timeout 300 python bench.py --workload n29 --no-cpu-baseline --steps 10 > gpurun_out/ab_n29.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_n29.json
done
