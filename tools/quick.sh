#!/bin/bash
# Quick GPU iteration: matern parity tests + M100 timing (+ optional ncu of one launch).
mkdir -p gpurun_out
TAG=${1:-q}
timeout 600 python -m pytest tests -m gpu -q -x -k "matern or edges or peer or smoke" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('M100 ms',round(d['value']*1e3,2),'clk',d['clocks'])"
if [ -n "$NCU" ]; then
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:matern_kernel -s 1 -c 1 -o gpurun_out/prof_matern_$TAG -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
echo "ncu rc=$?"
fi
