
CMD="python scripts/exp_one.py paper_1912_11494_b200/libsegb200.so 3 2"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_exp.csv $CMD > gpurun_out/ncu_exp.log 2>&1; echo ncu_rc=$?
