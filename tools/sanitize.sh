#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py,
# only this repo's kernels (mangled names containing "eca").  Logs in gpurun_out/.
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --kernel-name regex:eca --print-limit 50 \
    --log-file gpurun_out/sanitize_$tool.log python tools/sanitize_run.py > gpurun_out/sanitize_$tool.out 2>&1
  echo "$tool rc=$?"
  tail -3 gpurun_out/sanitize_$tool.log
done
