#!/bin/bash
# Round-2 session-2 validation: full GPU suite, bench, launch list (sampler after the per-group
# prune threshold).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g36_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g36_smoke.log
SART_PF_UMMA=0 timeout 600 python -m pytest -x -q -s tests/test_gpu_fullsize.py > gpurun_out/g36_fullsize_mma.log 2>&1; echo full_mma rc=$?; grep -a "logits row error" gpurun_out/g36_fullsize_mma.log
timeout 2400 python -m pytest tests -m gpu -x -q -s > gpurun_out/g36_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g36_pytest.log
timeout 900 python bench.py > gpurun_out/g36_bench.json 2> gpurun_out/g36_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/g36_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline']['with_merge']['frac'], d['step_roofline']['frac'], d['e2e']['value'], d['clocks'])"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 250000 -c 600 --csv --log-file gpurun_out/g36_launches.csv python tools/prof_c2.py --warm 3 --steps 0 > gpurun_out/g36_launches_run.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/g36_launches.csv > gpurun_out/g36_launch_list.txt 2>&1; head -16 gpurun_out/g36_launch_list.txt
