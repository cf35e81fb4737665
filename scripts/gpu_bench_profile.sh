set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc $?"
cat gpurun_out/bench_c4.json
python bench.py --workload n29 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n29.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n29.csv python bench.py --workload n29 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc $?"
python bench.py --workload n29 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n29b.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_stage -s 2 -c 2 -o gpurun_out/prof_n29 python bench.py --workload n29 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la gpurun_out
