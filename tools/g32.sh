#!/bin/bash
# Round-2 session-2 call 3: double-buffered P in the tcgen05 attention kernel (prefill / PRM
# pass / prefix pass), SART_ATTN_PIECE, IPC flake rate.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g32_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g32_smoke.log
timeout 1500 python -m pytest -x -q -s tests/test_gpu_parity.py -k "1p5b_shape or 7b_14b or long_prefix or prefix_tc or interleaved or pieces" > gpurun_out/g32_parity.log 2>&1; echo parity rc=$?
grep -a "worst\|passed\|failed\|Error" gpurun_out/g32_parity.log | tail -20
timeout 900 python -m pytest -x -q -s tests/test_gpu_prm_model.py > gpurun_out/g32_prm.log 2>&1; echo prm rc=$?; tail -1 gpurun_out/g32_prm.log
for u in 1 0; do
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 2>&1 | tail -1
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 1.5B --prompt 545 --requests 64 2>&1 | tail -1
done
for t in "0 64" "64 64" "64 96" "64 128"; do set -- $t
  SART_ATTN_TCQ=$1 SART_TC_SMS=$2 timeout 600 python tools/run_config.py --config c5 --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tcq=$1 sms=$2 c5', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'), d.get('attn_stream_frac_of_6455'), d.get('attn_ms_per_launch'))"
done
SART_ATTN_PIECE=128 timeout 1200 python -m pytest -x -q -s tests/test_gpu_fullsize.py > gpurun_out/g32_fullsize_p128.log 2>&1; echo full128 rc=$?
grep -a "logits row error\|passed\|failed" gpurun_out/g32_fullsize_p128.log | tail -3
for rep in 1 2; do for p in 0 128 64; do
  echo -n "piece=$p "; SART_ATTN_PIECE=$p timeout 600 python tools/ablate_c2.py --masks 0 2>&1 | tail -1
done; done
timeout 600 python -m pytest -x -q -s tests/test_gpu_tp.py -k ipc > gpurun_out/g32_ipc.log 2>&1; echo ipc rc=$?; grep -a "TP=2 IPC\|passed\|failed" gpurun_out/g32_ipc.log
for i in 1 2 3 4 5 6; do timeout 600 python tools/tp_ipc_debug.py 2>&1 | grep "rank 0 window 0 row b0"; done
timeout 900 python bench.py > gpurun_out/g32_bench.json 2> gpurun_out/g32_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/g32_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline']['with_merge']['frac'], d['step_roofline']['frac'], d['e2e']['value'])"
