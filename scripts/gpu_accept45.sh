# The reference's headline campaign (acceptance criteria 4 and 5: L = 9..18, 25 000
# problems x 256 shots, its own harness/acceptance code) on the B200 engine.
timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_dropin.py -x -q -p no:cacheprovider > gpurun_out/pytest_lock.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_lock.log
mkdir -p gpurun_out/acc
( time timeout 2400 oracle/_ref/acceptance_b200 --criterion 4 --criterion 5 --cache-dir gpurun_out/acc ) > gpurun_out/acceptance45.log 2>&1; echo "acceptance rc $?"
cat gpurun_out/acceptance45.log | tail -8
