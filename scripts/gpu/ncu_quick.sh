# one full ncu capture of k_classify and k_cull (exact mode) after the plain run exits 0: quick per-change check
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-stats"
timeout 600 $CMD > gpurun_out/plain_q.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_classify|k_cull" -s 6 -c 2 -o gpurun_out/prof_quick -f $CMD > gpurun_out/ncu_quick.log 2>&1; echo ncu_rc=$?
