#!/bin/bash
# N>1 launch check on one GPU: two ranks share cuda:0 (gloo for the host-side
# barrier/max), M100-shaped peer mode and BK, plus the reference arm under torchrun.
mkdir -p gpurun_out
export BGK_BENCH_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $R bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload m10 > gpurun_out/multi_m10.json 2> gpurun_out/multi_m10.err
echo "m10 peer rc=$?"; cat gpurun_out/multi_m10.json | head -c 700; echo
timeout 900 $R bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --workload bk > gpurun_out/multi_bk.json 2> gpurun_out/multi_bk.err
echo "bk rc=$?"; cat gpurun_out/multi_bk.json | head -c 400; echo
timeout 900 $R bench.py --impl reference --gpus 2 --steps 1 --warmup 3 --workload m10 > gpurun_out/multi_ref.json 2> gpurun_out/multi_ref.err
echo "ref rc=$?"; cat gpurun_out/multi_ref.json | head -c 300; echo
for w in m10 m50 m200; do
  timeout 900 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print(d['metric'],d['value'],d['ms_per_step'],d['cpu_baseline']['value'])"
done
