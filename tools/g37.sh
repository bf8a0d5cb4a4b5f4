#!/bin/bash
# cascade attention warp config A/B on C2 (in-graph step, alternating): 6 warps x 2 x 32 tokens (0)
# vs 7 warps x 2 x 32 (4, 224 KB of ring per SM)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2 3; do for c in 0 4; do
  echo -n "cfg=$c "; SART_ATTN_CFG=$c timeout 600 python tools/ablate_c2.py --masks 0 2>&1 | tail -1
done; done
for c in 0 4; do
  SART_ATTN_CFG=$c timeout 600 python tools/run_config.py --config c5 --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('cfg=$c c5', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_stream_frac_of_6455'), d.get('attn_ms_per_launch'))"
done
