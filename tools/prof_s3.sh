# Session-3 GPU profiling: ncu --set full of two mid-window cascade-attention launches in the
# bench workload (-> profiles/attn_traffic.json for roofline.traffic), and the launch list of
# one f2 PRM pass (C2 + PRM-7B, pass 2).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attn_cascade -s 39200 -c 2 -o gpurun_out/s3_attn_full python tools/attn_traffic.py --warm 3 > gpurun_out/attn_traffic_run.log 2>&1
ncu -i gpurun_out/s3_attn_full.ncu-rep --page raw --csv > gpurun_out/s3_attn_full.csv 2>/dev/null
python tools/attn_traffic.py --summarise gpurun_out/s3_attn_full.csv gpurun_out/attn_traffic_run.log > gpurun_out/s3_attn_traffic.json 2>&1
cp profiles/attn_traffic.json gpurun_out/attn_traffic.json
if [ -n "$PRM_LAUNCHES" ]; then
SART_NCU_PRM_PASS=2 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_prm_launches.csv python tools/run_config.py --config c2p --prm PRM-7B --warmup 1 --windows 1 > gpurun_out/s3_prm_ncu_run.log 2>&1
fi
cat gpurun_out/s3_attn_traffic.json
