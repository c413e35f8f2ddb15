# bench lines: default (N=1, cfg3), torchrun N=1, reference arm, FP32 peak probe
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp32_peak scripts/probes/fp32_peak.cu && /tmp/fp32_peak > gpurun_out/fp32_peak.txt 2>&1; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv >> gpurun_out/fp32_peak.txt
cat gpurun_out/fp32_peak.txt
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
python scripts/bench_brief.py gpurun_out/bench.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo torchrun_rc=$?
python scripts/bench_brief.py gpurun_out/bench_torchrun.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
cut -c1-600 gpurun_out/bench_ref.json
