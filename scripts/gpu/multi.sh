set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x 2>&1 | tail -3
python scripts/ab_build.py 3 ""
