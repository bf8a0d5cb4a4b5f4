#!/bin/bash
# TP IPC race hunt (default / no PDL / no graphs), sanitizer over the session-2 kernels, ncu of
# the tcgen05 causal prefill.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for mode in default SART_NO_PDL=1 SART_NO_GRAPHS=1; do
  for i in 1 2 3 4 5 6 7 8; do
    if [ $mode = default ]; then timeout 300 python tools/tp_ipc_debug.py 2>&1 | grep "rel err" | sed "s/^/$mode $i /"
    else env $mode timeout 300 python tools/tp_ipc_debug.py 2>&1 | grep "rel err" | sed "s/^/$mode $i /"; fi
  done
done > gpurun_out/g33_ipc.txt
awk '{bad=0; for(i=1;i<=NF;i++) if ($i ~ /e-0[0-1]$/ || $i ~ /e\+/) bad=1; print $1, bad}' gpurun_out/g33_ipc.txt | sort | uniq -c
grep -c . gpurun_out/g33_ipc.txt
SANITIZE_S2=1 bash tools/sanitize.sh 2>&1 | grep "s2" 
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_prefix_tc -s 40 -c 2 -o gpurun_out/g33_pf_umma \
  python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1 --reps 1 > gpurun_out/g33_pf_ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/g33_pf_umma.ncu-rep --page raw --csv > gpurun_out/g33_pf_umma.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/g33_pf_umma.csv')))
hdr=rows[0]
want=['gpu__time_duration.sum','sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active',
 'sm__throughput.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__bytes_write.sum','sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active',
 'smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    d=dict(zip(hdr,r))
    print(d.get('Kernel Name','')[:60], {k:d.get(k) for k in want if k in d})
tp=[h for h in hdr if 'tensor' in h.lower() and 'pct' in h.lower()]
print(tp[:20])
PY
