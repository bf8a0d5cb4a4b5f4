#!/bin/bash
# (1) tcgen05 causal kernel with two CTAs per SM (2 KV stages, one P buffer): parity + prefill A/B
# (2) cascade attention warp config A/B on C2 (6 x 2 x 32 vs 7 x 2 x 32)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/g37_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g37_smoke.log
timeout 1500 python -m pytest -x -q -s tests/test_gpu_parity.py -k "1p5b_shape or 7b_14b or long_prefix or prefix_tc or interleaved" > gpurun_out/g37_parity.log 2>&1; echo parity rc=$?
grep -a "worst\|passed\|failed\|Error" gpurun_out/g37_parity.log | tail -12
timeout 900 python -m pytest -x -q -s tests/test_gpu_prm_model.py > gpurun_out/g37_prm.log 2>&1; echo prm rc=$?; tail -1 gpurun_out/g37_prm.log
timeout 900 python -m pytest -x -q -s tests/test_gpu_fullsize.py > gpurun_out/g37_fullsize.log 2>&1; echo full rc=$?; grep -a "logits row error\|passed\|failed" gpurun_out/g37_fullsize.log | tail -2
for c2 in 1 0; do
  SART_PF_CTA2=$c2 timeout 300 python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 2>&1 | tail -1 | sed "s/^/cta2=$c2 /"
  SART_PF_CTA2=$c2 timeout 300 python tools/pf_bench.py --shape 1.5B --prompt 545 --requests 64 2>&1 | tail -1 | sed "s/^/cta2=$c2 /"
done
for rep in 1 2 3; do for c in 0 4; do
  echo -n "cfg=$c "; SART_ATTN_CFG=$c timeout 600 python tools/ablate_c2.py --masks 0 2>&1 | tail -1
done; done
