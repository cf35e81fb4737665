timeout 900 python -m pytest tests/test_dropin.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_dropin.log 2>&1; echo "dropin rc $?"; tail -2 gpurun_out/pytest_dropin.log
for c in 2 10 7 8 4 5; do
  timeout 1200 ./oracle/_ref/acceptance_b200 --criterion $c > gpurun_out/accept_b200_c$c.log 2>&1; echo "criterion $c rc $?"; tail -1 gpurun_out/accept_b200_c$c.log | cut -c1-400
done
