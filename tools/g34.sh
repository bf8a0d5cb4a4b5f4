#!/bin/bash
# after the init-ordering fix (dalloc zeroes on the ctx stream; legacy uploads device-synced):
# IPC pair x10, the TP suite, C3 / C5 with the prefix pass on by default.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g34_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g34_smoke.log
for i in 1 2 3 4 5 6 7 8 9 10; do timeout 300 python tools/tp_ipc_debug.py 2>&1 | grep "rank 0 rel err" | sed "s/^/$i /"; done | tee gpurun_out/g34_ipc.txt
timeout 900 python -m pytest -x -q -s tests/test_gpu_tp.py > gpurun_out/g34_tp.log 2>&1; echo tp rc=$?; grep -a "TP=\|passed\|failed" gpurun_out/g34_tp.log | tail -8
for c in c5 c3; do
  timeout 600 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('default $c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'), d.get('attn_stream_frac_of_6455'), d.get('attn_ms_per_launch'))"
done
