# 1) launch list of the default bench command (config 4), after a clean run of the same command
python bench.py > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc $?"
# 2) full captures of the tiled probs and collapse kernels at the n29 profiling size
CMD="python bench.py --workload n29 --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_n29_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_finalize" -s 0 -c 4 -o gpurun_out/prof_v5_n29 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
tail -2 gpurun_out/ncu_full.log
