#!/bin/bash
# per-test durations of the GPU suite (the round-end step has a 20-minute limit)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SART_LONG_GPU_TESTS=1 timeout 3000 python -m pytest tests -m gpu -q --durations=0 > gpurun_out/g41_durations.log 2>&1; echo rc=$?
grep -a "s call\|s setup\|passed\|failed" gpurun_out/g41_durations.log | head -80
