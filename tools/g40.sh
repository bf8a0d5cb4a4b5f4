#!/bin/bash
# C5 / C3 with the prefix on the tensor-core pass: is a shorter attention chunk (more suffix
# items than the 888 warps) better now?
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ch in 512 256 512 256; do for c in c5 c3; do
  SART_ATTN_CH=$ch timeout 600 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ch=$ch $c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_stream_frac_of_6455'), d.get('attn_ms_per_launch'))"
done; done
