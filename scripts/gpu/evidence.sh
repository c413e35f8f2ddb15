# round evidence at HEAD: smoke, GPU suite (with the oracle cache: every-fiber parity), full-size parity report,
# the default bench line, the reference arm, the per-config report
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/smoke.log
timeout 2400 python scripts/full_parity.py > gpurun_out/full_parity.log 2>&1; echo parity_rc=$?; tail -1 gpurun_out/full_parity.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -5
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python scripts/bench_brief.py gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
timeout 1500 python scripts/report.py > gpurun_out/report_rows.jsonl 2> gpurun_out/report.err; echo report_rc=$?
timeout 900 python scripts/bench_rows.py 3 > gpurun_out/bench_rows.jsonl 2> gpurun_out/bench_rows.err; echo rows_rc=$?
