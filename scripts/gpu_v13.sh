# v13: pooled lockstep buffers + attribute queries at create: GPU tests, create cost, headline campaign
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_v13.log 2>&1; echo "pytest rc $?"; tail -1 gpurun_out/pytest_v13.log
python scripts/create_cost.py; python scripts/create_cost.py
mkdir -p gpurun_out/acc
( time timeout 2400 oracle/_ref/acceptance_b200 --criterion 4 --criterion 5 --cache-dir gpurun_out/acc ) > gpurun_out/acceptance45_v13.log 2>&1; echo "acceptance rc $?"
tail -7 gpurun_out/acceptance45_v13.log
