# speculative write in the direct kernels too: the whole GPU suite, smoke, the default bench, c3 timing
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/v16_bench_c4.json 2> gpurun_out/v16_bench_c4.err; echo "bench rc $?"; tail -2 gpurun_out/v16_bench_c4.err
python scripts/summarize_bench.py gpurun_out/v16_bench_c4.json | cut -c1-600
for sp in 1 0; do echo "SHS_SPEC=$sp"; SHS_SPEC=$sp timeout 300 python scripts/c3_time.py 2>&1 | head -2; SHS_SPEC=$sp python scripts/lock_profile.py 1048573 3; done
