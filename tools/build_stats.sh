#!/bin/bash
# diagnostic build of libeca with ECA_STATS counters -> build/libeca_stats.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build/stats
for f in paper_2210_14771_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DECA_STATS -Xcompiler -fPIC -Iinclude -c "$f" -o build/stats/$(basename $f .cu).o
done
g++ -O2 -std=c++17 -fPIC -Iinclude -c paper_2210_14771_b200/csrc/eca_host.cpp -o build/stats/eca_host.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/libeca_stats.so build/stats/*.o
