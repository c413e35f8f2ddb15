# e2e repeatability: the host-buffer path of cfg 3 measured in 4 separate processes, with the NUMA layout
set -x
nvidia-smi topo -m; lscpu | grep -i numa
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
for i in 1 2 3 4; do timeout 600 python bench.py --steps 5 --warmup 3 --no-stats --no-cpu-baseline --e2e-steps 10 > gpurun_out/e2e_$i.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/e2e_$i.json').read().splitlines()[-1]); print('run $i ms/step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],2))"; done
python scripts/probes/h2d_bw.py
