#!/bin/bash
# L2 evict-first policy on the suffix KV stream of the cascade attention: C2 in-graph step A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2 3; do for e in 0 1; do
  echo -n "evict=$e "; SART_ATTN_EVICT=$e timeout 600 python tools/ablate_c2.py --masks 0 2>&1 | tail -1
done; done
for e in 0 1; do
  SART_ATTN_EVICT=$e timeout 600 python tools/run_config.py --config c3 --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('evict=$e c3', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_stream_frac_of_6455'), d.get('attn_frac_of_6455'))"
done
