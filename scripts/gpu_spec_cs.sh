# A/B: evict-first (st.global.cs) speculative h0 stores (variants/lib_speccs.so) vs plain
for rep in 1 2; do
for lib in variants/lib_speccs.so paper_2308_05047_b200/libshorsim_b200.so; do
SHS_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-small > gpurun_out/ab.json 2>/dev/null; python -c "
import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1])
print('$lib', round(d['ms_per_step'],3), {k:(round(v['avg_ms'],3),v['launches']) for k,v in d['kernels'].items()}, 's/run', round(d['s_per_run'],3), 'dense', round(d['s_per_run_dense'],3), d['clocks']['reasons'])"
done; done
