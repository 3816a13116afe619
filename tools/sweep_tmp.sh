python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/prof_kernels.py 256 2>&1 | grep -E "points.2|pipelined|engine"
cp tools/alt/lib_128.so paper_2210_14771_b200/libeca_b200.so
echo "128 regs: $(python tools/prof_kernels.py 256 2>&1 | grep -E 'pipelined')"
cp tools/alt/lib_times.so paper_2210_14771_b200/libeca_b200.so
python tools/warp_times.py 2>&1 | head -8
