# round-2 measurement recipe: bench (N=1), launch list and one-kernel full ncu capture at config 4
set -x
mkdir -p gpurun_out/r02
python -c "import sys; sys.path.insert(0,'.'); from oracle import reference_build; print(reference_build())"
grep -m1 'model name' /proc/cpuinfo; nproc
python bench.py > gpurun_out/r02/bench_c4.json 2> gpurun_out/r02/bench_c4.err; echo "bench rc $?"
tail -3 gpurun_out/r02/bench_c4.err
python bench.py --impl reference > gpurun_out/r02/bench_reference.json 2>&1; echo "ref rc $?"
CMD="python bench.py --steps 4 --warmup 3 --no-small --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02/launches_c4.csv $CMD > gpurun_out/r02/ncu_launch.log 2>&1; echo "ncu launches rc $?"
ncu --set full --clock-control none --import-source on -k regex:k_tiled -s 4 -c 2 -o gpurun_out/r02/prof_c4_ktiled $CMD > gpurun_out/r02/ncu_full.log 2>&1; echo "ncu full rc $?"
ls -la gpurun_out/r02
