#!/bin/bash
# A/B two builds of libsart on the C2 bench, interleaved: tools/ab_lib.sh "libA.so libB.so" [rounds]
# build a variant with: SART_LIB_OUT=$PWD/build_ab/x.so SART_NVCC_EXTRA="-DFOO=1" python paper_2505_13326_b200/build.py
LIBS=$1; R=${2:-2}
for r in $(seq $R); do for l in $LIBS; do
  SART_LIB=$l timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $l)', round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['frac'],3))"
done; done
