#!/bin/bash
# A/B of the GEMM split choice on small-M configs (C70, C5, C3) and the C2 bench.
for lib in "$@"; do
  n=$(basename $lib)
  for c in ${CONFIGS:-c70 c5 c3}; do
    SART_LIB=$lib timeout 600 python tools/run_config.py --config $c --warmup 1 --windows 2 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', '$c', round(d['branch_tokens_per_s'],1), round(d['ms_per_decode_step'],2))"
  done
  [ -n "$NOBENCH" ] || SART_LIB=$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', 'c2-bench', round(d['value']), round(d['ms_per_step'],1))"
done
