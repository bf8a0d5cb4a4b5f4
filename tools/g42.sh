#!/bin/bash
# the round-end GPU steps as the driver runs them (default tier; the step limit is 20 minutes)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
start=$(date +%s); timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/g42_pytest.log 2>&1; echo pytest rc=$? seconds=$(( $(date +%s) - start ))
tail -3 gpurun_out/g42_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
