timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "small_multiplier or tiled or tile_plans" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_q.log
timeout 300 python scripts/c3_breakdown.py 4294967213 5 > gpurun_out/c4_bd.log 2>&1; head -2 gpurun_out/c4_bd.log | cut -c1-160; tail -5 gpurun_out/c4_bd.log
timeout 600 python bench.py --no-cpu-baseline --no-small --steps 8 > gpurun_out/ab_c4.json 2>&1 && python scripts/summarize_bench.py gpurun_out/ab_c4.json | cut -c1-200
