# SURVEY.md Sec. 8(d) report: bench lines for configs 0-4 x both modes, CPU oracle timings on the host cores
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
timeout 1500 python scripts/report.py > gpurun_out/report_rows.jsonl 2> gpurun_out/report.err; echo report_rc=$?
timeout 900 python scripts/cpu_report.py > gpurun_out/cpu_report.jsonl 2> gpurun_out/cpu_report.err; echo cpu_rc=$?
wc -l gpurun_out/report_rows.jsonl gpurun_out/cpu_report.jsonl
