#!/bin/bash
# compute-sanitizer memcheck over the smallest end-to-end paths: smoke (C1 control + logits)
# and the f2 PRM-model pass (tiny policy + prm-tiny, bf16 and fp32).
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" \
  > gpurun_out/sanitize_smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/sanitize_smoke.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_prm_model.py -x -q \
  -k "tiny-prm-tiny-bf16-16-40-None or tiny-prm-tiny-fp32-16-40-100" > gpurun_out/sanitize_f2.log 2>&1; echo f2_rc=$?; tail -3 gpurun_out/sanitize_f2.log
# shared-memory races and barrier misuse on the same small paths
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_prm_model.py -x -q \
    -k "tiny-prm-tiny-bf16-16-40-None" > gpurun_out/sanitize_$tool.log 2>&1; echo ${tool}_rc=$?; tail -2 gpurun_out/sanitize_$tool.log
done
# memcheck over the small-shape decode parity (cascade attention, tcgen05 GEMMs, sampler, prefill)
# and the on-device control traces
if [ -n "$SANITIZE_DECODE" ]; then
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_control.py -x -q \
  -k "tiny_bf16 or small_gqa or sampler or trace_A or trace_B or random_scripted_workloads[0] or tight_pool[16-4]" \
  > gpurun_out/sanitize_decode.log 2>&1; echo decode_rc=$?; tail -3 gpurun_out/sanitize_decode.log
fi
# round 2: memcheck over the new device paths -- the interleaved prefill schedule, es_every_step,
# record_trace replay, the CTA-pair GEMM and a caller-owned KV pool.  The TP exchange is not run
# here: its ranks spin on each other's arrivals, which needs concurrent kernels, and the
# sanitizer serialises launches (the 20 s watchdog in k_tp_wait would trap).
if [ -n "$SANITIZE_R2" ]; then
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_control.py \
  tests/test_gpu_replay.py tests/test_gpu_gemm.py tests/test_gpu_api.py -x -q \
  -k "interleaved_prefill_random_workloads[0] or es_every_step_trace_B or model_mode_bf16_replay[True] or cta_pair_matches_one_sm[200 or kv_pool" \
  > gpurun_out/sanitize_r2.log 2>&1; echo r2_rc=$?; tail -3 gpurun_out/sanitize_r2.log
fi
# round 2, session 2: the tcgen05 attention kernel in its three modes (causal prefill of the
# hd-128 `small` shape, the concurrent prefix pass, the f2 PRM pass over prm-small) and the
# suffix pieces (SART_ATTN_PIECE)
if [ -n "$SANITIZE_S2" ]; then
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prm_model.py -x -q \
  -k "prefix_tc_pass[small or pieces[small or small-prm-small-bf16" > gpurun_out/sanitize_s2.log 2>&1; echo s2_rc=$?; tail -3 gpurun_out/sanitize_s2.log
for tool in racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_prm_model.py -x -q \
    -k "small-prm-small-bf16-16-40-None" > gpurun_out/sanitize_s2_$tool.log 2>&1; echo s2_${tool}_rc=$?; tail -2 gpurun_out/sanitize_s2_$tool.log
done
fi
