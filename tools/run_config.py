"""Run one BASELINE.json configuration on one GPU and print a JSON line.

    python tools/run_config.py --config c3 --windows 4 --warmup 2

c1: tiny decoder, 1 request, N=4, M=2, cap 64, T=16, alpha 0.5, beta 2 (BJ configs[0])
c3: 7B shape, 32 requests/GPU (the per-GPU share of 256 on 8 GPUs), N=16, M=4, cap 8192,
    T=400, alpha 0.5, beta 8, scripted rewards (BJ configs[2]); admission is commitment-limited
c70: the paper's 70B model shape on ONE B200 (TP = 1; row f4's TP split: tools/run_tp.py),
    16 requests (commitment admits ~66 rows at a time, the rest queue), N=8, M=4, cap 2048, alpha 0.5, beta 4
c5: 14B shape, 8192-token shared prompt, N=32, M=16, alpha 0.5, beta 16, cap 16384, T=400,
    1 request per GPU (BJ configs[4])
c2p: C2's workload (1.5B, 64 requests, N=8, M=4, cap 4096, T=400) with PRM pruning
    (alpha 0.5, beta 4) scored by a separate PRM decoder (row f2): --prm PRM-7B is the
    Qwen2.5-Math-PRM-7B shape.  Scripted lengths, PRM-model scores.
Values: branch-tokens/s over the timed windows (CUDA events), attention roofline over one
extra eager window (same method as bench.py); with --prm also the PRM pass GPU time per
boundary and its tensor-pipe rate (2 x matmul params x entries read, attention flops excluded).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CONFIGS = {
    "c1": dict(shape="tiny", n_req=1, N=4, M=2, alpha=0.5, beta=2, cap=64, T=16, p=(16, 16), B=64, bs=16),
    "c3": dict(shape="7B", n_req=32, N=16, M=4, alpha=0.5, beta=8, cap=8192, T=400, p=(64, 1024), B=1024, bs=64),
    "c2p": dict(shape="1.5B", n_req=64, N=8, M=4, alpha=0.5, beta=4, cap=4096, T=400, p=(64, 1024), B=512, bs=64),
    # the paper's 70B model on one GPU (TP = 1): N=8, M=4, cap 2048 (the ~30 GB pool left
    # after 141 GB of weights commits ~40 rows of 2048 tokens), scripted lengths and rewards
    "c70": dict(shape="70B", n_req=16, N=8, M=4, alpha=0.5, beta=4, cap=2048, T=400, p=(64, 1024), B=512, bs=64),
    "c5": dict(shape="14B", n_req=1, N=32, M=16, alpha=0.5, beta=16, cap=16384, T=400, p=(8193, 8193), B=64, bs=64),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--windows", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--prm", default=None, help="separate PRM decoder shape (row f2), e.g. PRM-7B")
    ap.add_argument("--requests", type=int, default=0, help="override the config's request count")
    ap.add_argument("--num-blocks", type=int, default=0, help="KV pool blocks (0: from free HBM; ncu needs room)")
    a = ap.parse_args()
    import torch
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_requests
    c = dict(CONFIGS[a.config])
    if a.requests:
        c["n_req"] = a.requests
    shape = SHAPES[c["shape"]]
    prm = None
    if a.prm:   # the PRM reads the policy's tokens: give it the policy's vocab
        import dataclasses
        prm = dataclasses.replace(SHAPES[a.prm], vocab=shape.vocab)
    stream = torch.cuda.current_stream()
    t0 = time.time()
    eng = Engine(shape, "bf16", weight_seed=3, block_size=c["bs"], num_blocks=a.num_blocks, max_rows=c["B"], max_requests=256,
                 max_prompt=c["p"][1] + 1, T=c["T"], cap=c["cap"], eos_id=1, temperature=1.0, sampler_seed=5,
                 stream=stream.cuda_stream, prm_shape=prm, prm_weight_seed=11)
    init_s = time.time() - t0
    reqs = gen_requests(c["n_req"], shape, c["N"], c["M"], c["alpha"], c["beta"], c["cap"], c["T"], eos_id=1,
                        p_range=c["p"])
    for r in reqs:
        eng.admit(r, use_script_scores=prm is None)     # with a PRM model its scores drive pruning
    if a.config == "c1":      # latency config: time the whole request (no warm-up)
        a.warmup, a.windows = 0, 1000
    t0 = time.time()
    eng.step(a.warmup)
    torch.cuda.synchronize()
    warm_s = time.time() - t0
    s0, p0 = eng.step(0), eng.profile()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.step(a.windows)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    s1, p1 = eng.step(0), eng.profile()
    eng.set_profile(2)     # events around the attention operator and between its two kernels
    q0 = eng.profile()
    eng.step(1)
    torch.cuda.synchronize()
    q1 = eng.profile()
    eng.set_profile(False)
    att_ms, att_b = q1["attn_ms"] - q0["attn_ms"], q1["attn_bytes"] - q0["attn_bytes"]
    st = eng.step(0)
    out = {"config": a.config, "shape": c["shape"], "windows_timed": s1["windows"] - s0["windows"],
           "decode_steps": s1["steps"] - s0["steps"],
           "branch_tokens_per_s": (s1["branch_tokens"] - s0["branch_tokens"]) / (ms / 1e3),
           "requests_finalized": s1["finalized_total"] - s0["finalized_total"], "ms_timed": ms,
           "ms_per_decode_step": ms / max(1, s1["steps"] - s0["steps"]),
           "us_per_decode_step": 1e3 * ms / max(1, s1["steps"] - s0["steps"]),
           "prefill_ms_timed": p1["prefill_ms"] - p0["prefill_ms"],
           "live_rows_end": st["live_rows"], "queued_requests_end": st["queued_requests"],
           "free_blocks": st["free_blocks"], "committed_blocks": st["committed_blocks"],
           "attn_GBps": att_b / (att_ms / 1e3) / 1e9 if att_ms else None,
           "attn_frac_of_6455": att_b / (att_ms / 1e3) / 1e9 / 6455.3 if att_ms else None,
           "attn_ms_per_launch": att_ms / max(1, q1["attn_launches"] - q0["attn_launches"]),
           "attn_stream_frac_of_6455": att_b / ((q1["attn_stream_ms"] - q0["attn_stream_ms"]) / 1e3) / 1e9 / 6455.3
           if q1["attn_stream_ms"] > q0["attn_stream_ms"] else None,
           "init_s": init_s, "warmup_s": warm_s}
    if prm is not None:
        d, F, L = prm.d_model, prm.d_ff, prm.n_layers
        params = L * (d * prm.qkv_dim + d * prm.n_heads * prm.head_dim + 3 * d * F) + d * d
        passes = p1["prm_passes"] - p0["prm_passes"]
        pms, ptok = p1["prm_ms"] - p0["prm_ms"], p1["prm_tokens"] - p0["prm_tokens"]
        out.update({"prm_shape": a.prm, "prm_passes": passes, "prm_ms_per_pass": pms / max(1, passes),
                    "prm_share_of_timed": pms / ms, "prm_entries_per_s": ptok / (pms / 1e3) if pms else None,
                    "prm_matmul_TFLOPs": 2.0 * params * ptok / (pms / 1e3) / 1e12 if pms else None,
                    "prm_frac_of_1385_TFLOPs": 2.0 * params * ptok / (pms / 1e3) / 1e12 / 1385.5 if pms else None,
                    "pruned_total": None})
        res = eng.collect()
        out["pruned_total"] = sum(r["num_pruned"] for r in res)
        out["early_stopped_total"] = sum(r["num_early_stopped"] for r in res)
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
