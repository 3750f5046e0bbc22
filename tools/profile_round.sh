#!/bin/bash
# ncu evidence for profiles/: full captures of the two hot kernels + the bench launch list.
set -x
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:matern_kernel -s 1 -c 1 \
     -o gpurun_out/prof_matern -f python tools/profile_kernels.py matern 20000 1.5 > gpurun_out/ncu_matern.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:besselk_kernel -s 1 -c 1 \
     -o gpurun_out/prof_besselk -f python tools/profile_kernels.py besselk 16777216 > gpurun_out/ncu_besselk.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ls -la gpurun_out
