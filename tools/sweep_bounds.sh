#!/bin/bash
# bound-and-prune launch shape sweep: register cap x warps per CTA
for reg in 80 96 112 128; do
  ECA_NVCC_DEFINES="-DECA_BOUNDS_MAXREG=$reg" python -m paper_2210_14771_b200.build --force > /dev/null || exit 1
  for w in 0 1 2 4 8; do
    echo -n "maxreg $reg warps/CTA ${w} (0 = auto): "
    ECA_BWARPS=$w python tools/time_bounds_pdl.py 2>&1 | tail -1
  done
done
python -m paper_2210_14771_b200.build --force > /dev/null
