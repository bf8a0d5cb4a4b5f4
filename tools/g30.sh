#!/bin/bash
# Round-2 session-2 HEAD validation: build, smoke, full GPU suite, default bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g30_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/g30_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g30_pytest.log
timeout 900 python bench.py > gpurun_out/g30_bench.json 2> gpurun_out/g30_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/g30_bench.json
