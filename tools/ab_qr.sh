#!/bin/bash
# prefix-group size (branches per cascade prefix group) A/B on C5, C3 and the C2 bench
for qr in default 32; do
  if [ $qr = default ]; then E=""; else E="SART_ATTN_QR=$qr"; fi
  for c in c5 c3; do
    env $E timeout 600 python tools/run_config.py --config $c --warmup 1 --windows 2 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('QR=$qr', '$c', round(d['branch_tokens_per_s'],1), round(d['ms_per_decode_step'],2), round(d['attn_frac_of_6455'],3))"
  done
  env $E timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('QR=$qr', 'c2', round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['frac'],3))"
done
