# speculative group-0 write: parity (full GPU suite) and the config-4 A/B (SHS_SPEC=0 = every collapse runs)
python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "speculative or forced or tiled or c4_size or seeded" > gpurun_out/pytest_spec.log 2>&1; echo "pytest spec rc $?"; tail -3 gpurun_out/pytest_spec.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/spec_on.json 2> gpurun_out/spec_on.err; echo "bench on rc $?"; tail -2 gpurun_out/spec_on.err
SHS_SPEC=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/spec_off.json 2> gpurun_out/spec_off.err; echo "bench off rc $?"
for f in spec_on spec_off; do python -c "
import json,sys;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step'],3), d['stage_bytes_per_amp'], round(d['stage_frac_of_hbm'],3), d['speculative_group0'], {k:(round(v['avg_ms'],3),v['launches']) for k,v in d['kernels'].items()}, 's/run', round(d['s_per_run'],3), 'dense', round(d['s_per_run_dense'],3), d['clocks'])"; done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest all rc $?"; tail -3 gpurun_out/pytest_gpu.log
