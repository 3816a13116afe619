#!/bin/bash
# One GPU call's worth of round evidence, written under gpurun_out/:
# GPU tests, smoke, the default bench line, the ncu launch list of a short
# bench, ncu --set full of the dominant kernel (bounds_kernel) and of the
# tensor-core CNN.   usage: tools/round_capture.sh TAG
tag=${1:-r}
o=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $o/${tag}_tests.log 2>&1; echo "tests_rc=$?" >> $o/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1
timeout 900 python bench.py > $o/${tag}_bench.json 2> $o/${tag}_bench.err; echo "bench_rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $o/${tag}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > $o/${tag}_ncu_list.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bounds_kernel -s 2 -c 1 \
  -o $o/${tag}_bounds python tools/ncu_target.py points > $o/${tag}_ncu_bounds.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cnn_kernel_tc -c 1 \
  -o $o/${tag}_cnn python tools/ncu_learned.py > $o/${tag}_ncu_cnn.log 2>&1
echo done
