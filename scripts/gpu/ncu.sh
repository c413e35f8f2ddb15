# ncu evidence (B200_PROFILING.md recipe): the launch list of a short bench run, then one --set full capture of
# k_classify (exact and paper mode) and of k_cull, each after the same command exited 0 without ncu
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
timeout 600 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_classify -s 3 -c 1 -o gpurun_out/prof_classify -f $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_cull -s 3 -c 1 -o gpurun_out/prof_cull -f $CMD > gpurun_out/ncu_cull.log 2>&1; echo cull_rc=$?
PCMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mode paper"
timeout 600 $PCMD > gpurun_out/plain3.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_classify -s 3 -c 1 -o gpurun_out/prof_classify_paper -f $PCMD > gpurun_out/ncu_full_paper.log 2>&1; echo full_paper_rc=$?
ls -la gpurun_out/*.ncu-rep
