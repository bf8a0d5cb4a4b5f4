#!/bin/bash
# C5 attention DRAM traffic with the concurrent tensor-core prefix pass (single-pass metrics:
# the 14B pool leaves ncu no room to back up device memory for replays)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
W5=2; L5=48
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_read.sum \
  --clock-control none -k regex:"k_attn_(cascade|prefix_tc)" -s $(( (W5*400+200)*L5*2 )) -c 8 --csv --page raw \
  --log-file gpurun_out/g47_c5_attn.csv \
  python tools/attn_traffic.py --config c5 --warm $W5 --num-blocks 8400 > gpurun_out/g47_c5_attn.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/g47_c5_attn.log
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/g47_c5_attn.csv')))
hdr=None
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); print(d['Kernel Name'][:40], d.get('Metric Name'), d.get('Metric Value'), d.get('Metric Unit'))
PY
