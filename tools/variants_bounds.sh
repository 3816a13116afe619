#!/bin/bash
# Rebuild with each -D set; time the bound-and-prune kernel (pipeline launch
# mode and isolated) and the pipelined step.   usage: tools/variants_bounds.sh "DEFS1" ...
for defs in "$@"; do
  ECA_NVCC_DEFINES="$defs" python -m paper_2210_14771_b200.build --force > /dev/null || exit 1
  echo "== $defs"
  timeout 120 python tools/time_bounds_pdl.py 2>&1 | tail -1
  QUICK=1 timeout 120 python tools/prof_bounds.py 256 2>&1 | tail -1
done
python -m paper_2210_14771_b200.build --force > /dev/null
