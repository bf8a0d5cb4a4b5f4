#!/bin/bash
# A/B of attention variants at an identical C2 state (window 4, step 1, layers 0..2) under ncu
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active"
for merge in 0 1; do for cfg in 0 1 2; do
  SART_ATTN_MERGE=$merge SART_ATTN_CFG=$cfg SART_NO_GRAPHS=1 timeout 600 ncu --metrics $M --clock-control none --cache-control none -k regex:"k_attn_(cascade|merge)" -s $((33600*(2-merge))) -c $((6-3*merge)) --csv --log-file gpurun_out/ab_${merge}_${cfg}.csv python tools/prof_c2.py --warm 3 --steps 1 > /dev/null 2>&1
  python - "$merge" "$cfg" <<'PY'
import csv, sys, collections
m, c = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(f"gpurun_out/ab_{m}_{c}.csv")))
hdr = [r for r in rows if "Kernel Name" in r][0]
vals = collections.defaultdict(list)
for r in rows:
    if len(r) == len(hdr) and r != hdr:
        d = dict(zip(hdr, r)); k = d["Kernel Name"].split("(")[0].split("::")[-1][:22]
        vals[(k, d["Metric Name"])].append(float(d["Metric Value"].replace(",", "")))
out = {k: sum(v) / len(v) for k, v in vals.items()}
print("merge", m, "cfg", c, {f"{k[0]}:{k[1].split('__')[1][:14]}": round(v, 2) for k, v in sorted(out.items())})
PY
done; done
