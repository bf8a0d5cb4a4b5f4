#!/bin/bash
# tcgen05 causal prefill (f1) + concurrent tensor-core prefix pass: parity, then A/B; TP flake debug.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g31_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/g31_smoke.log
timeout 600 python tools/tp_flaky.py > gpurun_out/g31_tp_flaky.log 2>&1; echo tpflaky rc=$?; grep -v "^$" gpurun_out/g31_tp_flaky.log | tail -12
for i in 1 2; do timeout 600 python tools/tp_ipc_debug.py 2>&1 | grep "rel err"; done
timeout 1200 python -m pytest -x -q -s tests/test_gpu_parity.py -k "1p5b or 7b_14b or long_prefix or prefix_tc or interleaved or production_ch" > gpurun_out/g31_parity.log 2>&1; echo parity rc=$?
grep -a "worst\|passed\|failed\|Error" gpurun_out/g31_parity.log | tail -20
timeout 900 python -m pytest -x -q -s tests/test_gpu_prm_model.py > gpurun_out/g31_prm.log 2>&1; echo prm rc=$?; tail -2 gpurun_out/g31_prm.log
for u in 0 1; do
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 1.5B --prompt 545 --requests 64 2>&1 | tail -1
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 2>&1 | tail -1
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 7B --prompt 2049 --requests 8 2>&1 | tail -1
done
timeout 900 python bench.py > gpurun_out/g31_bench.json 2> gpurun_out/g31_bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/g31_bench.json')); print(d['value'], d['roofline']['frac'], d['roofline']['with_merge']['frac'], d['step_roofline']['frac'], d['e2e']['value'])"
for c in c5 c3; do for t in "0 64" "64 32" "64 64" "64 96"; do set -- $t
  SART_ATTN_TCQ=$1 SART_TC_SMS=$2 timeout 600 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tcq=$1 sms=$2 $c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'), d.get('attn_stream_frac_of_6455'), d.get('attn_ms_per_launch'), d.get('prefill_ms_timed'))"
done; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 250000 -c 600 --csv --log-file gpurun_out/g31_launches.csv python tools/prof_c2.py --warm 3 --steps 0 > gpurun_out/g31_launches_run.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/g31_launches.csv > gpurun_out/g31_launch_list.txt 2>&1; head -25 gpurun_out/g31_launch_list.txt
