#!/bin/bash
# build variants (ECA_NVCC_DEFINES), each timed with tools/time_pipe.py
for d in "$@"; do
  echo "== $d"
  ECA_NVCC_DEFINES="$d" python -m paper_2210_14771_b200.build --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python tools/time_pipe.py 2>&1 | grep -E "steps=200|bounds only" | grep -v "ready=False"
done
