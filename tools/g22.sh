timeout 600 python -m pytest -x -q -s tests/test_gpu_parity.py -k "prefix_tc_pass or long_prefix" > gpurun_out/tc_tests.log 2>&1; echo rc=$?
grep -a "prefix tc\|long prefix\|passed\|failed\|Error\|error" gpurun_out/tc_tests.log | head -30
for c in c5 c3; do for t in 64 0; do
  SART_ATTN_TCQ=$t timeout 600 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tcq=$t $c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'), d.get('attn_ms_per_launch'))"
done; done
for e in "SART_GEMM_2SM=0" "SART_QKV_HALF=0" "SART_GEMM_2SM=2"; do
  env $e SART_ATTN_TCQ=0 timeout 600 python tools/run_config.py --config c3 --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$e c3', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3))"
done
