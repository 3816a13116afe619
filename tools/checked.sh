#!/bin/bash
# ECA_CHECKED build (device-side index checks trap) + the sanitizer workload +
# the GPU parity suite; then the normal build again.  Logs in gpurun_out/.
set -u
mkdir -p gpurun_out
ECA_NVCC_DEFINES=-DECA_CHECKED python -m paper_2210_14771_b200.build --force > gpurun_out/checked_build.log 2>&1 || exit 1
python tools/sanitize_run.py > gpurun_out/checked_workload.log 2>&1; echo "checked workload rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/checked_tests.log 2>&1
echo "checked gpu tests rc=$?"; tail -2 gpurun_out/checked_tests.log
python -m paper_2210_14771_b200.build --force > /dev/null 2>&1
