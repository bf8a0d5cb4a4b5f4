#!/bin/bash
# final: default tier as the driver runs it, smoke, bench, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
start=$(date +%s); timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/g44_pytest.log 2>&1; echo pytest rc=$? seconds=$(( $(date +%s) - start ))
tail -2 gpurun_out/g44_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/g44_bench.json 2> gpurun_out/g44_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/g44_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline']['with_merge']['frac'], d['step_roofline']['frac'], d['e2e']['value'], d['clocks'])"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 250000 -c 600 --csv --log-file gpurun_out/g44_launches.csv python tools/prof_c2.py --warm 3 --steps 0 > gpurun_out/g44_launches_run.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/g44_launches.csv > gpurun_out/g44_launch_list.txt 2>&1; head -12 gpurun_out/g44_launch_list.txt
