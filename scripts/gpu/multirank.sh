# functional check of bench.py's multi-rank paths on ONE GPU: 2 and 3 ranks on cuda:0 over gloo (strong and weak)
set -x
python -c "from paper_1912_11494_b200 import _build; _build.build(force=True)"
export SEG_BENCH_ONE_DEVICE=1 SEG_BENCH_BACKEND=gloo
for n in ${MR_N:-2 3}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --gpus $n --steps 3 --warmup 3 --e2e-steps 2 --no-stats > gpurun_out/mr_strong_$n.json 2> gpurun_out/mr_strong_$n.err; echo strong_${n}_rc=$?
  tail -c 1500 gpurun_out/mr_strong_$n.json; tail -5 gpurun_out/mr_strong_$n.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29529 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 2 --no-stats --scaling weak --config 2 > gpurun_out/mr_weak_2.json 2> gpurun_out/mr_weak_2.err; echo weak_rc=$?
tail -c 1500 gpurun_out/mr_weak_2.json; tail -5 gpurun_out/mr_weak_2.err
for n in ${MR_N:-2 3}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 3 --warmup 3 --e2e-steps 2 --no-stats --gather p2p > gpurun_out/mr_p2p_$n.json 2> gpurun_out/mr_p2p_$n.err; echo p2p_${n}_rc=$?
  tail -c 1200 gpurun_out/mr_p2p_$n.json; tail -5 gpurun_out/mr_p2p_$n.err
done
timeout 900 python -m pytest tests/test_gpu_p2p_gather.py -q -p no:cacheprovider 2>&1 | tail -5
