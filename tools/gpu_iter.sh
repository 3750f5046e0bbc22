#!/bin/bash
# One GPU iteration: parity tests, a quick bench (no e2e / CPU leg), ncu captures of both
# hot kernels.  Writes everything under gpurun_out/.
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -2 gpurun_out/bench_$TAG.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench_$TAG.json"))
print("M100 s", round(d["value"], 5), "frac", round(d["roofline"]["frac"], 3), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
s = d["secondary"]; print("BK evals/s %.4g" % s["value"], "frac", round(s["roofline"]["frac"], 3), "ms", round(s["ms_per_step"], 4))
PY
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:matern_kernel -s 1 -c 1 -o gpurun_out/prof_matern_$TAG -f python tools/profile_kernels.py matern 20000 1.5 > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:besselk_kernel -s 1 -c 1 -o gpurun_out/prof_besselk_$TAG -f python tools/profile_kernels.py besselk 16777216 > /dev/null 2>&1
echo "ncu done"
