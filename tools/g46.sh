#!/bin/bash
# ncu --set full of two mid-window k_attn_cascade launches in the bench workload (final build:
# suffix KV with the L2 evict-first policy) -> profiles/attn_traffic.json (roofline.traffic)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_attn_cascade -s 39200 -c 2 -o gpurun_out/g46_attn_full python tools/attn_traffic.py --warm 3 > gpurun_out/g46_attn_run.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/g46_attn_full.ncu-rep --page raw --csv > gpurun_out/g46_attn_full.csv 2>/dev/null
python tools/attn_traffic.py --summarise gpurun_out/g46_attn_full.csv gpurun_out/g46_attn_run.log > gpurun_out/g46_attn_traffic.json 2>&1
cp profiles/attn_traffic.json gpurun_out/g46_attn_traffic_profiles.json
cat gpurun_out/g46_attn_traffic.json
ncu -i gpurun_out/g46_attn_full.ncu-rep --page details --csv 2>/dev/null | grep -a "k_attn_cascade" | awk -F'","' '{print $(NF-3)" | "$(NF-2)" | "$(NF-1)" | "$NF}' | grep -E "Duration|DRAM Throughput|Memory Throughput|SM Active|L2 Hit|Issued Ipc|Eligible" | head -20 > gpurun_out/g46_attn_summary.txt
cat gpurun_out/g46_attn_summary.txt
