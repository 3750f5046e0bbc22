#!/bin/bash
# A/B for the BesselK kernel: rebuild with -D flags, time the 64Mi BK batch, one ncu capture each.
mkdir -p gpurun_out
i=0
for V in "$@"; do
  i=$((i+1))
  make -s -C paper_2502_00356_b200 -B EXTRA="$V" > /dev/null 2>&1 || { echo "build failed for $V"; continue; }
  python bench.py --workload bk --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/abk.json 2>/dev/null
  T=$(python -c "import json;d=json.load(open('gpurun_out/abk.json'));print(round(d['ms_per_step'],4),'ms', '%.4g evals/s'%d['value'])")
  /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:besselk_kernel -s 1 -c 1 -o gpurun_out/abk_$i -f python tools/profile_kernels.py besselk 16777216 > /dev/null 2>&1
  echo "[$i: $V] BK $T"
done
make -s -C paper_2502_00356_b200 -B > /dev/null 2>&1
