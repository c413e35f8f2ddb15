timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log | grep -v Warn
for c in 1 3 4; do timeout 600 python scripts/exp_seed.py $c ; done
