#!/bin/bash
# A/B: rebuild the library with different -D flags on the box and time M100 + ncu each.
mkdir -p gpurun_out
for V in "$@"; do
  make -s -C paper_2502_00356_b200 -B EXTRA="$V" > /dev/null 2>&1 || { echo "build failed for $V"; continue; }
  python bench.py --no-e2e --no-cpu-baseline --no-secondary --steps 3 > gpurun_out/ab.json 2>/dev/null
  T=$(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']*1e3,2),'ms frac',round(d['roofline']['frac'],3))")
  TAG=$(echo "$V" | tr -c 'A-Za-z0-9' '_')
  /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:matern_kernel -s 1 -c 1 -o gpurun_out/ab_$TAG -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
  echo "[$V] M100 $T"
done
make -s -C paper_2502_00356_b200 -B > /dev/null 2>&1
