timeout 300 python -m pytest -q tests/test_gpu_api.py -k kv_pool > gpurun_out/kvpool.log 2>&1; tail -2 gpurun_out/kvpool.log
for c in c1 c3 c5 c70; do timeout 900 python tools/run_config.py --config $c --warmup 2 --windows 3 2>/dev/null | tail -1 >> gpurun_out/r2_configs.jsonl; done; cat gpurun_out/r2_configs.jsonl | cut -c1-300
SANITIZE_R2=1 bash tools/sanitize.sh 2>&1 | tail -15
