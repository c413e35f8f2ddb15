# ad-hoc experiment runner: EXP_CMD is a ;-separated list of commands
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
eval "${EXP_CMD}"
