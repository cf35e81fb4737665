# Full ncu captures of the lockstep kernels at N = 262139 (one launch each, past
# the warm-up run), then the reference's headline campaign (acceptance 4 + 5).
mkdir -p gpurun_out/acc
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lock_probs -s 60 -c 1 -o gpurun_out/prof_lock_probs -f python scripts/lock_profile.py 262139 4242 > gpurun_out/ncu_lock_probs.log 2>&1; echo "ncu probs rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lock_collapse -s 60 -c 1 -o gpurun_out/prof_lock_collapse -f python scripts/lock_profile.py 262139 4242 > gpurun_out/ncu_lock_collapse.log 2>&1; echo "ncu collapse rc $?"
( time timeout 2400 oracle/_ref/acceptance_b200 --criterion 4 --criterion 5 --cache-dir gpurun_out/acc ) > gpurun_out/acceptance45_v12.log 2>&1; echo "acceptance rc $?"
tail -8 gpurun_out/acceptance45_v12.log
