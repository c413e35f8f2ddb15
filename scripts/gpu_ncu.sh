# launch list + one full capture of the classify kernel (B200_PROFILING.md recipe)
set -x
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_classify -s 3 -c 1 -o gpurun_out/prof_classify $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
