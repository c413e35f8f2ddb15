# quick evidence at HEAD: the default bench line, the launch list, one full capture of k_classify and k_cull
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python scripts/bench_brief.py gpurun_out/bench.json
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
bash scripts/gpu/ncu_quick.sh
