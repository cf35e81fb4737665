timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider > gpurun_out/pytest_mp.log 2>&1; echo "mp rc $?"; tail -5 gpurun_out/pytest_mp.log
SHS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload n29 --steps 4 --warmup 3 > gpurun_out/bench_2rank_n29.json 2> gpurun_out/bench_2rank_n29.err; echo "2-rank bench rc $?"
tail -c 1500 gpurun_out/bench_2rank_n29.json; tail -5 gpurun_out/bench_2rank_n29.err
