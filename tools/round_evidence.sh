#!/bin/bash
# Round evidence in one call: full default bench line (e2e + CPU baseline), the
# reference arm, ncu launch list of the bench command, full-size DRAM traffic of both
# hot kernels, and one ncu --set full capture of each hot kernel.
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 1200 python bench.py > gpurun_out/bench_full_$TAG.json 2> gpurun_out/bench_full_$TAG.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref rc=$?"
bash tools/profile_traffic.sh
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:matern_kernel -s 1 -c 1 \
     -o gpurun_out/prof_matern_$TAG -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:besselk_kernel -s 1 -c 1 \
     -o gpurun_out/prof_besselk_$TAG -f python tools/profile_kernels.py besselk 16777216 > /dev/null 2>&1
echo "ncu done"
