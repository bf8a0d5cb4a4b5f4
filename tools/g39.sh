#!/bin/bash
# Session-2 final validation: smoke, full GPU suite, bench, C1 / C3 / C5 single-GPU runs, launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g39_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g39_smoke.log
timeout 2700 python -m pytest tests -m gpu -x -q -s > gpurun_out/g39_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/g39_pytest.log
timeout 900 python bench.py > gpurun_out/g39_bench.json 2> gpurun_out/g39_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/g39_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline']['with_merge']['frac'], d['step_roofline']['frac'], d['e2e']['value'], d['clocks'])"
for c in c1 c3 c5; do timeout 900 python tools/run_config.py --config $c --warmup 2 --windows 3 2>/dev/null | tail -1; done > gpurun_out/g39_configs.jsonl; cat gpurun_out/g39_configs.jsonl | cut -c1-300
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 250000 -c 600 --csv --log-file gpurun_out/g39_launches.csv python tools/prof_c2.py --warm 3 --steps 0 > gpurun_out/g39_launches_run.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/g39_launches.csv > gpurun_out/g39_launch_list.txt 2>&1; head -14 gpurun_out/g39_launch_list.txt
