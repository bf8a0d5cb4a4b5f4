#!/bin/bash
# small-M gate/up: split-K GEMM + SwiGLU-over-partials (1) vs the fused SwiGLU GEMM (0), C5
for r in 1 2; do for v in 0 1; do
  SART_SWIGLU_SPLIT=$v timeout 600 python tools/run_config.py --config c5 --warmup 1 --windows 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SWIGLU_SPLIT=$v c5', round(d['branch_tokens_per_s'],1), round(d['ms_per_decode_step'],2))"
done; done
