#!/bin/bash
# A/B prebuilt library variants on one box: usage bash tools/ab_libs.sh [--bk] ab/libA.so ab/libB.so ...
# (build them here first, e.g. tools/build_variant.sh).  Each variant is swapped in
# as the package library and timed (M100, or the BK batch with --bk), twice, interleaved.
mkdir -p gpurun_out
LIB=paper_2502_00356_b200/libbesselgp_sm100a.so
cp $LIB /tmp/lib_orig.so
WL="--no-secondary"
if [ "$1" == "--bk" ]; then WL="--workload bk"; shift; fi
if [ "$1" == "--wl" ]; then WL="--workload $2 --no-secondary"; shift 2; fi
for rep in 1 2; do
  for V in "$@"; do
    cp "$V" $LIB
    python bench.py --no-e2e --no-cpu-baseline $WL --steps 5 > gpurun_out/ab.json 2>/dev/null
    T=$(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['ms_per_step'],3),'ms clk',d['clocks']['sm_mhz'])")
    echo "[$rep $V] $T"
  done
done
cp /tmp/lib_orig.so $LIB
