# e2e repeatability for one config / mode (report.py showed occasional slow e2e lines)
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
for i in 1 2 3; do timeout 600 python bench.py --config ${CFG:-2} --mode ${MODE:-paper} --steps 5 --warmup 3 --no-stats --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2ev_$i.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/e2ev_$i.json').read().splitlines()[-1]); print('run $i', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2))"; done
