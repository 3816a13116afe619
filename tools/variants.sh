#!/bin/bash
# Rebuild libeca_b200.so with each -D set and time the bound-and-prune kernel
# and the pipelined step (tools/prof_bounds.py).  usage: tools/variants.sh "DEFS1" "DEFS2" ...
for defs in "$@"; do
  ECA_NVCC_DEFINES="$defs" python -m paper_2210_14771_b200.build --force > /dev/null || exit 1
  echo "== $defs"
  QUICK=1 python tools/prof_bounds.py 256 2>&1 | grep -v "^$"
done
python -m paper_2210_14771_b200.build --force > /dev/null
