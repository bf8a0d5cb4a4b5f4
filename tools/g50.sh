#!/bin/bash
# the gpu_long tier on the final build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SART_LONG_GPU_TESTS=1 timeout 2400 python -m pytest tests -m gpu_long -x -q -s > gpurun_out/g50_long.log 2>&1; echo rc=$?
grep -a "worst\|PP3\|TP=\|passed\|failed" gpurun_out/g50_long.log | tail -14
