mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_peer.py tests/test_distributed.py -q -x 2>&1 | tail -3
export BGK_BENCH_BACKEND=gloo
for G in 2 4; do
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $G --master-addr 127.0.0.1 --master-port 2953$G"
timeout 900 $R bench.py --gpus $G --steps 2 --warmup 3 --no-cpu-baseline --workload m10 > gpurun_out/multi_m10_g$G.json 2> gpurun_out/multi_m10_g$G.err
echo "m10 G=$G rc=$?"; head -c 900 gpurun_out/multi_m10_g$G.json; echo
done
