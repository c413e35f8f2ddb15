# parity tests + a short bench + stats (no ncu)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -4 gpurun_out/pytest_gpu.log | grep -v Warning
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python scripts/bench_brief.py gpurun_out/bench.log
timeout 300 python scripts/stats_cfg.py 3 > gpurun_out/stats3.log 2>&1; tail -1 gpurun_out/stats3.log | cut -c1-1500
