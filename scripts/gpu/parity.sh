# full-size parity (every fiber, configs 0-4, both modes) + the GPU suite with the oracle cache present
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
nproc
timeout 2400 python scripts/full_parity.py > gpurun_out/full_parity.log 2>&1; echo parity_rc=$?
tail -3 gpurun_out/full_parity.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | head -30
