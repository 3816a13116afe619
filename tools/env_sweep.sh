#!/bin/bash
# runtime env variants, each timed with tools/time_pipe.py (steady state lines)
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/time_pipe.py 2>&1 | grep -E "steps=200|bounds only|run_stream 20 steps, pause 0.0" | grep -v "ready=False"
done
