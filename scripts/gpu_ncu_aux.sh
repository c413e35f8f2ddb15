# one full ncu capture of each auxiliary kernel (prepass + k_cull), first timed launch of bench.py
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_cull|k_morton|k_scan" -s 12 -c 4 -o gpurun_out/prof_aux -f $CMD > gpurun_out/ncu_aux.log 2>&1; echo aux_rc=$?
tail -2 gpurun_out/ncu_aux.log
