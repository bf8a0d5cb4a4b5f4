#!/bin/bash
# SART_TC_PAIR=1 (8 softmax warps, two per row, bit-identical arithmetic): parity, prefill + C5 A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export SART_TC_PAIR=1
timeout 900 python -m pytest -x -q -s tests/test_gpu_parity.py -k "1p5b_shape or 7b_14b or long_prefix or prefix_tc or interleaved" > gpurun_out/g48_parity.log 2>&1; echo parity rc=$?
grep -a "worst\|passed\|failed\|Error" gpurun_out/g48_parity.log | tail -9
timeout 600 python -m pytest -x -q tests/test_gpu_prm_model.py > gpurun_out/g48_prm.log 2>&1; echo prm rc=$?; tail -1 gpurun_out/g48_prm.log
timeout 600 python -m pytest -x -q -s tests/test_gpu_fullsize.py > gpurun_out/g48_full.log 2>&1; echo full rc=$?; grep -a "logits row error" gpurun_out/g48_full.log
for pr in 1 0; do
  SART_TC_PAIR=$pr timeout 300 python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 2>&1 | tail -1 | sed "s/^/pair=$pr /"
  SART_TC_PAIR=$pr timeout 600 python tools/run_config.py --config c5 --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('pair=$pr c5', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_stream_frac_of_6455'))"
done
