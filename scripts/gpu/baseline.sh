set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_base.log 2>&1; echo bench_rc=$?
python scripts/bench_brief.py gpurun_out/bench_base.log
for c in 1 2 4; do timeout 600 python scripts/ab_build.py $c "" ; done
