#!/bin/bash
# A/B of the prefill / PRM-pass attention variants on the f2 workload (C2 + PRM-7B):
# prints prm_ms_per_pass and branch-tok/s per variant.
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python tools/run_config.py --config c2p --prm PRM-7B --warmup 1 --windows 2 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', round(d['prm_ms_per_pass'],1), round(d['branch_tokens_per_s']), round(d['prefill_ms_timed'],1))"
}
run ungrouped SART_PF_GROUP=0
run grouped_nst4
run grouped_minb2_nst3 SART_LIB=$PWD/build_ab/minb2.so SART_PF_NST=3
run grouped_minb2_nst2 SART_LIB=$PWD/build_ab/minb2.so SART_PF_NST=2
run ungrouped SART_PF_GROUP=0
