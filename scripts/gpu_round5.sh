timeout 120 python scripts/tiled_smoke.py > gpurun_out/tiled_smoke.log 2>&1; rc=$?; echo "tiled smoke rc $rc"
if [ $rc -ne 0 ]; then tail gpurun_out/tiled_smoke.log; exit 1; fi
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -4 gpurun_out/pytest_gpu.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc $?"
python scripts/summarize_bench.py gpurun_out/bench_c4.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc $?"
CMD="python bench.py --workload n29 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_n29_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile" -s 0 -c 3 -o gpurun_out/prof_r32_n29 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
tail -1 gpurun_out/ncu_full.log
