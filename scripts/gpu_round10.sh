# v10 profile set (final kernels): default bench, reference arm, launch list,
# full ncu captures at n30 (tiled round-robin kernels, fixup, measure; sparse-prefix kernels).
timeout 900 python bench.py > gpurun_out/v10_bench_c4.json 2> gpurun_out/v10_bench_c4.err; echo "bench rc $?"
python scripts/summarize_bench.py gpurun_out/v10_bench_c4.json | cut -c1-400
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/v10_bench_reference.json 2> gpurun_out/v10_ref.err; echo "ref rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/v10_launches_c4.csv python bench.py --no-cpu-baseline --no-small > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc $?"
CMD="python bench.py --workload n30 --steps 3 --warmup 3 --no-cpu-baseline --no-small"
$CMD > gpurun_out/v10_bench_n30.json 2>&1; echo "n30 plain rc $?"; python scripts/summarize_bench.py gpurun_out/v10_bench_n30.json | cut -c1-300
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tiled|k_tile_fixup|k_finalize" -c 6 -o gpurun_out/prof_v10_n30 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc $?"; tail -1 gpurun_out/ncu_full.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_sparse_(expand|fold|collapse)" -s 66 -c 3 -o gpurun_out/prof_v10_sparse_n30 $CMD > gpurun_out/ncu_sparse.log 2>&1; echo "ncu sparse rc $?"; tail -1 gpurun_out/ncu_sparse.log
