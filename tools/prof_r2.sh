#!/bin/bash
# Round-2 ncu captures (one GPU, under gpurun).  Outputs land in gpurun_out/.
#  1. C2: the decode GEMMs (QKV half-head, O, gate/up, down) mid-window, --set full
#  2. C2: the cascade attention kernel mid-window, --set full (DRAM bytes vs algorithmic)
#  3. C5: the cascade attention kernel mid-window, single-pass DRAM metrics (the 105 GB pool
#     + 28 GB of weights leave ncu no room to back up device memory for replays)
set -x
W=3; L=28
# QKV (half-head tiles <64, 4, 1>) launches are only decode launches: skip W windows + half a window
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_gemm_tc<\\(int\\)64, \\(int\\)4" -s $(( (W*400+200)*L )) -c 2 -o gpurun_out/r2_qkv \
  python tools/attn_traffic.py --config c2 --warm $W > gpurun_out/r2_qkv.log 2>&1
# one layer's O / gate-up / down GEMMs right after a QKV launch mid-window: capture 12 GEMM
# launches (prefill launches make the skip approximate; the grid sizes identify each kernel)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"k_gemm_tc<\\(int\\)(128, \\(int\\)0|256, \\(int\\)2|256, \\(int\\)0)" -s $(( (W*400+200)*L*3 )) -c 6 -o gpurun_out/r2_gemms \
  python tools/attn_traffic.py --config c2 --warm $W > gpurun_out/r2_gemms.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_attn_(cascade|merge)" -s $(( (W*400+200)*L*2 )) -c 4 -o gpurun_out/r2_attn \
  python tools/attn_traffic.py --config c2 --warm $W > gpurun_out/r2_attn.log 2>&1
W5=2; L5=48
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum \
  --clock-control none -k regex:k_attn_cascade -s $(( (W5*400+200)*L5 )) -c 6 --csv --page raw \
  --log-file gpurun_out/r2_c5_attn.csv \
  python tools/attn_traffic.py --config c5 --warm $W5 --num-blocks 8400 > gpurun_out/r2_c5_attn.log 2>&1
ls -la gpurun_out/
