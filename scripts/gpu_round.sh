# round evidence: tests, smoke, bench (default args), launch list + one full ncu capture of k_classify
set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches_rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_classify -s 3 -c 1 -o gpurun_out/prof_classify -f $CMD > gpurun_out/ncu_full.log 2>&1; echo full_rc=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k_cull -s 3 -c 1 -o gpurun_out/prof_cull -f $CMD > gpurun_out/ncu_cull.log 2>&1; echo cull_rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo torchrun_rc=$?
timeout 600 python scripts/bench_rows.py 3 > gpurun_out/bench_rows.jsonl 2> gpurun_out/bench_rows.err; echo rows_rc=$?
timeout 900 python bench.py --mode paper --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_paper.json 2> gpurun_out/bench_paper.err; echo paper_rc=$?
