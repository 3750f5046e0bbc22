#!/bin/bash
# Quick GPU iteration on the Matern kernel: parity tests, an M100 timing (no e2e /
# CPU legs) and one ncu --set full capture of the kernel.  usage: bash tools/quick.sh TAG [--bk]
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_matern.py tests/test_parity_edges.py tests/test_full_size.py tests/test_api_gpu.py tests/test_preprocess_gp.py tests/test_peer.py tests/test_kernel_geometry.py -m gpu -x -q > gpurun_out/quick_pytest_$TAG.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/quick_pytest_$TAG.log)"
for w in m100 m50; do
  timeout 600 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-secondary --steps 5 > gpurun_out/quick_${w}_$TAG.json 2> gpurun_out/quick_${w}_$TAG.err
  python -c "import json;d=json.load(open('gpurun_out/quick_${w}_$TAG.json'));r=d['roofline'];print('$w', round(d['ms_per_step'],3),'ms frac',r.get('frac'),'clk',d['clocks']['sm_mhz'])"
done
X="--metrics sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.sum"
/usr/local/cuda/bin/ncu --set full $X --clock-control none --import-source on -k regex:matern_kernel -s 1 -c 1 \
     -o gpurun_out/prof_matern_$TAG -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
echo "ncu rc=$?"
