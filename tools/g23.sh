timeout 1500 python -m pytest -x -q -s tests/test_gpu_parity.py tests/test_gpu_fullsize.py > gpurun_out/swap_tests.log 2>&1; echo rc=$?
grep -a "logits row\|worst\|passed\|failed\|Error" gpurun_out/swap_tests.log | tail -30
for i in 1 2; do python tools/ablate_c2.py --masks 0 2>&1 | tail -1; done
for c in c5 c3; do
  timeout 600 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1 | \
  python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'), d.get('attn_ms_per_launch'))"
done
