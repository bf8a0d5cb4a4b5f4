#!/bin/bash
# Phase timestamps (CTA 0) of C2 decode GEMM launches: build variants with -DSART_GEMM_TS
# -DSART_GEMM_TS_MODE=<mode> under build_ab/, then run one eager window per variant.
for v in $*; do
  SART_LIB=$PWD/build_ab/$v.so SART_GEMM_TS_PRINT=1 timeout 300 python tools/attn_traffic.py --config c2 --warm 2 2>&1 | grep GEMMTS | tail -8
done
