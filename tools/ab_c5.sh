#!/bin/bash
# C5 (14B, 8K shared prompt, N=32) under attention chunk-size / config overrides.
for ch in ${CHS:-512 1024 2048}; do for cfg in ${CFGS:-0 2}; do
  SART_ATTN_CH=$ch SART_ATTN_CFG=$cfg timeout 600 python tools/run_config.py --config c5 --warmup 1 --windows 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('CH=$ch CFG=$cfg', round(d['branch_tokens_per_s'],1), round(d['ms_per_decode_step'],2), round(d['attn_frac_of_6455'],3), round(d['attn_ms_per_launch']*1e3,1))"
done; done
