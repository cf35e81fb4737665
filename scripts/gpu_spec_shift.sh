# speculative h0 stores: sector-shifted (tree) vs plain (variants/lib_specplain.so); parity of the shifted stores first
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "speculative or forced or tiled or c4_size or seeded" > gpurun_out/pytest_spec.log 2>&1; echo "pytest spec rc $?"; tail -1 gpurun_out/pytest_spec.log
for rep in 1 2; do
for lib in variants/lib_specplain.so paper_2308_05047_b200/libshorsim_b200.so; do
SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-small > gpurun_out/ab.json 2>/dev/null; python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', round(d['ms_per_step'],3), d['stage_bytes_per_amp'], round(d['stage_frac_of_hbm'],3), {k:(round(v['avg_ms'],3),v['launches']) for k,v in d['kernels'].items()}, 's/run', round(d['s_per_run'],3), 'dense', round(d['s_per_run_dense'],3), d['clocks']['reasons'])"
done; done
CMD="python bench.py --workload n30 --steps 3 --warmup 3 --no-cpu-baseline --no-small"
for lib in variants/lib_specplain.so paper_2308_05047_b200/libshorsim_b200.so; do
echo "== ncu $lib"; SHS_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_tiled<1" -c 2 $CMD 2>/dev/null | grep -E "k_tiled|duration|bytes" | head -8
done
