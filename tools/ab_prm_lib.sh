#!/bin/bash
# A/B two builds on the f2 workload (C2 + PRM-7B): prm_ms_per_pass, branch-tok/s, prefill ms
for r in 1 2; do for lib in "$@"; do
  SART_LIB=$lib timeout 600 python tools/run_config.py --config c2p --prm PRM-7B --warmup 1 --windows 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', round(d['prm_ms_per_pass'],1), round(d['branch_tokens_per_s']), round(d['prefill_ms_timed'],1))"
done; done
