# Full round trip on the restored tree: smoke, GPU parity tests, default bench
# (with the CPU baseline), its launch list, and full ncu captures at n29.
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -12 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc $?"
python scripts/summarize_bench.py gpurun_out/bench_c4.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc $?"; tail -c 600 gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --no-cpu-baseline --no-small > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc $?"
CMD="python bench.py --workload n29 --steps 3 --warmup 3 --no-cpu-baseline --no-small"
$CMD > gpurun_out/bench_n29_plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_finalize|k_stage" -s 0 -c 6 -o gpurun_out/prof_v8_n29 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
tail -2 gpurun_out/ncu_full.log
