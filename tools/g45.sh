#!/bin/bash
# L2 evict-first policy on the tcgen05 GEMMs' weight tiles (SART_GEMM_EVICT): C2 in-graph step A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2 3; do for e in 0 1; do
  echo -n "gemm_evict=$e "; SART_GEMM_EVICT=$e timeout 600 python tools/ablate_c2.py --masks 0 2>&1 | tail -1
done; done
for e in 0 1; do
  SART_GEMM_EVICT=$e timeout 600 python tools/run_config.py --config c3 --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('gemm_evict=$e c3', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3))"
done
