#!/bin/bash
# Quick GPU iteration for the BesselK kernel: parity tests + BK timing (+ optional ncu).
mkdir -p gpurun_out
TAG=${1:-q}
timeout 600 python -m pytest tests -m gpu -q -x -k "besselk or api or smoke or audit" > gpurun_out/pytest_bk_$TAG.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_bk_$TAG.log
timeout 300 python bench.py --workload bk --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/bench_bk_$TAG.json 2> gpurun_out/bench_bk_$TAG.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_bk_$TAG.json'));print('BK evals/s %.4g'%d['value'],'ms',round(d['ms_per_step'],4),'clk',d['clocks'])"
if [ -n "$NCU" ]; then
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:besselk_kernel -s 1 -c 1 -o gpurun_out/prof_besselk_$TAG -f python tools/profile_kernels.py besselk 16777216 > /dev/null 2>&1
echo "ncu rc=$?"
fi
