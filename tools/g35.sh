#!/bin/bash
# tcgen05 attention softmax fast path (unmasked tiles without predicates, ex2.approx, 8 max /
# 4 sum chains): parity of the three modes, prefill A/B, C3 / C5, ncu of the prefill kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g35_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g35_smoke.log
timeout 1500 python -m pytest -x -q -s tests/test_gpu_parity.py -k "1p5b_shape or 7b_14b or long_prefix or prefix_tc or interleaved" > gpurun_out/g35_parity.log 2>&1; echo parity rc=$?
grep -a "worst\|passed\|failed\|Error" gpurun_out/g35_parity.log | tail -14
timeout 900 python -m pytest -x -q -s tests/test_gpu_prm_model.py > gpurun_out/g35_prm.log 2>&1; echo prm rc=$?; tail -1 gpurun_out/g35_prm.log
timeout 1200 python -m pytest -x -q -s tests/test_gpu_fullsize.py > gpurun_out/g35_fullsize.log 2>&1; echo full rc=$?; grep -a "logits row error\|passed\|failed" gpurun_out/g35_fullsize.log | tail -2
for u in 1 0; do
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 2>&1 | tail -1
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 1.5B --prompt 545 --requests 64 2>&1 | tail -1
  SART_PF_UMMA=$u timeout 300 python tools/pf_bench.py --shape 7B --prompt 2049 --requests 8 2>&1 | tail -1
done
for t in "0 96" "64 64" "64 96"; do set -- $t
  for c in c5 c3; do
  SART_ATTN_TCQ=$1 SART_TC_SMS=$2 timeout 600 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tcq=$1 sms=$2 $c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'), d.get('attn_stream_frac_of_6455'), d.get('attn_ms_per_launch'))"
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_prefix_tc -s 140 -c 2 -o gpurun_out/g35_pf_umma \
  python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 --reps 1 > gpurun_out/g35_pf_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/g35_pf_umma.ncu-rep --page details --csv 2>/dev/null | grep -a "Duration\|Issued Ipc\|Executed Instructions\"\|SM Active\|Tensor" | head -12
