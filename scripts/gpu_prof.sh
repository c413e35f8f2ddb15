timeout 600 python scripts/exp_seed.py 3
CMD="python scripts/exp_one.py paper_1912_11494_b200/libsegb200.so 3 2"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_classify -s 1 -c 1 -o gpurun_out/prof_classify -f $CMD > gpurun_out/ncu_exp.log 2>&1; echo ncu_rc=$?
