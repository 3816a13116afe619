#!/bin/bash
# Rebuild with each -D set and time K4 (tools/time_mask.py).  usage: tools/variants_mask.sh "DEFS1" ...
for defs in "$@"; do
  ECA_NVCC_DEFINES="$defs" python -m paper_2210_14771_b200.build --force > /dev/null || exit 1
  echo "== $defs"
  python tools/time_mask.py
done
python -m paper_2210_14771_b200.build --force > /dev/null
