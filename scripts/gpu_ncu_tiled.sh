CMD="python bench.py --workload n29 --steps 4 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/bench_n29_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_finalize" -s 0 -c 4 -o gpurun_out/prof_ldgsts_n29 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc $?"
tail -2 gpurun_out/ncu_full.log
