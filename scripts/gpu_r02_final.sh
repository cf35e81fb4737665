# round-2 final measurement: full GPU suite, bench (N=1), reference arm, 2-rank
# bench (ranks sharing the GPU), launch list and one-kernel ncu at config 4
set -x
mkdir -p gpurun_out/r02f
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02f/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/r02f/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f/smoke.log 2>&1; echo "smoke rc $?"
python bench.py > gpurun_out/r02f/bench_c4.json 2> gpurun_out/r02f/bench_c4.err; echo "bench rc $?"
python bench.py --impl reference > gpurun_out/r02f/bench_reference.json 2>&1; echo "ref rc $?"
SHS_BENCH_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --workload n30 --steps 3 --warmup 3 > gpurun_out/r02f/bench_2ranks_n30.json 2> gpurun_out/r02f/bench_2ranks.err; echo "2rank rc $?"
SHS_X2_ROUNDS=2 timeout 900 python scripts/x2_probe.py n31 4 > gpurun_out/r02f/x2_probe_n31_g4.json 2>&1; echo "probe rc $?"
ls -la gpurun_out/r02f
