# one full ncu capture of k_cull (first timed launch of bench.py), with source
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_cull -s 3 -c 1 -o gpurun_out/prof_cull -f $CMD > gpurun_out/ncu_cull.log 2>&1; echo cull_rc=$?
tail -2 gpurun_out/ncu_cull.log
