#!/bin/bash
# DRAM traffic of the full-size hot launches (single-pass metrics: no kernel replay of
# the 80 GB output) + the launch list of the default bench command.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
$NCU --metrics $M --clock-control none -k regex:matern_kernel -s 2 -c 1 --csv \
     --log-file gpurun_out/traffic_m100.csv python tools/profile_kernels.py matern 100000 1.5 > /dev/null 2>&1
echo "m100 rc=$?"
$NCU --metrics $M --clock-control none -k regex:besselk_kernel -s 2 -c 1 --csv \
     --log-file gpurun_out/traffic_bk.csv python tools/profile_kernels.py besselk 67108864 > /dev/null 2>&1
echo "bk rc=$?"
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
     python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo "launches rc=$?"
