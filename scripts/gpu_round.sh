# GPU round trip: parity tests, c4 bench (+CPU baseline), n29 bench, then one ncu --set full
# capture of the tiled kernels on the n29 profiling size (after its plain run exited 0).
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc $?"
python scripts/summarize_bench.py gpurun_out/bench_c4.json
CMD="python bench.py --workload n29 --steps 6 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_n29.json 2> gpurun_out/bench_n29.err && python scripts/summarize_bench.py gpurun_out/bench_n29.json && \
ncu --set full --clock-control none --import-source on -k regex:k_tile -s 0 -c 3 -o gpurun_out/prof_tiled_n29 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/ncu_full.log
