#!/bin/bash
# Round evidence in one gpurun call (one GPU):
#   1. the default bench line (e2e, cpu_baseline, secondary BK lines, scalar latency)
#   2. the reference arm as the driver runs it (--steps 20 --warmup 5)
#   3. ncu launch list of a short bench command (gpu__time_duration, clocks untouched)
#   4. one ncu --set full capture per hot kernel (+ the FP64-pipe instruction count)
#   5. full-size single-pass DRAM traffic of both hot kernels
# then `python tools/evidence.py TAG` (here, after the call) writes profiles/.
# usage: bash tools/evidence.sh TAG [--no-bench] [--no-ref]
TAG=${1:-r02}; shift
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
if [[ " $* " != *" --no-bench "* ]]; then
  timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
  echo "bench rc=$?"
fi
if [[ " $* " != *" --no-ref "* ]]; then
  timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err
  echo "ref rc=$?"
fi
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
     python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu_$TAG.log 2>&1
echo "launches rc=$?"
X="--metrics sm__inst_executed_pipe_fp64.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.sum"
$NCU --set full $X --clock-control none --import-source on -k regex:matern_kernel -s 1 -c 1 \
     -o gpurun_out/prof_matern_$TAG -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
echo "ncu matern rc=$?"
$NCU --set full $X --clock-control none --import-source on -k regex:besselk_kernel -s 1 -c 1 \
     -o gpurun_out/prof_besselk_$TAG -f python tools/profile_kernels.py besselk 16777216 > /dev/null 2>&1
echo "ncu besselk rc=$?"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
$NCU --metrics $M --clock-control none -k regex:matern_kernel -s 2 -c 1 --csv \
     --log-file gpurun_out/traffic_m100_$TAG.csv python tools/profile_kernels.py matern 100000 1.5 > /dev/null 2>&1
echo "traffic m100 rc=$?"
$NCU --metrics $M --clock-control none -k regex:besselk_kernel -s 2 -c 1 --csv \
     --log-file gpurun_out/traffic_bk_$TAG.csv python tools/profile_kernels.py besselk 67108864 > /dev/null 2>&1
echo "traffic bk rc=$?"
