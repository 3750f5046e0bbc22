#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over every kernel
# (tools/sanitize_kernels.py); logs under gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
timeout 300 python tools/sanitize_kernels.py > gpurun_out/sanitize_plain.log 2>&1
echo "plain rc=$?"; tail -2 gpurun_out/sanitize_plain.log
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $T --error-exitcode 9 python tools/sanitize_kernels.py > gpurun_out/sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/sanitize_$T.log
done
