#!/bin/bash
# A/B: rebuild the library with different -D flags on the box, time M100 and take
# one ncu capture (N=20K launch) per variant.  usage: bash tools/ab_matern.sh "" "-DX=1" ...
mkdir -p gpurun_out
i=0
for V in "$@"; do
  i=$((i+1))
  make -s -C paper_2502_00356_b200 -B EXTRA="$V" > /dev/null 2>&1 || { echo "build failed for $V"; continue; }
  python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 3 > gpurun_out/ab.json 2>/dev/null
  T=$(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']*1e3,2),'ms clk',d['clocks']['sm_mhz'])")
  /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:matern_kernel -s 1 -c 1 -o gpurun_out/ab_$i -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
  echo "[$i: $V] M100 $T"
done
make -s -C paper_2502_00356_b200 -B > /dev/null 2>&1
