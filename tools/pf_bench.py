"""Prefill throughput (row f1): admit K requests with P-token prompts into an empty engine and
time the batched prefill of the first window (CUDA events around the fill loop's prefill,
sart_profile.prefill_ms).  A/B the attention kernel with SART_PF_UMMA=0 (mma.sync) vs the
default (tcgen05).  Prints one JSON line per (shape, P, K).

    python tools/pf_bench.py --shape 1.5B --prompt 544 --requests 64
    python tools/pf_bench.py --shape 14B --prompt 8193 --requests 1
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1.5B")
    ap.add_argument("--prompt", type=int, default=544)
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--num-blocks", type=int, default=0)
    a = ap.parse_args()
    import torch
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_requests
    shape = SHAPES[a.shape]
    stream = torch.cuda.current_stream()
    eng = Engine(shape, "bf16", weight_seed=3, block_size=64, num_blocks=a.num_blocks, max_rows=max(64, 8 * a.requests),
                 max_requests=max(8, a.requests), max_prompt=a.prompt + 1, T=1, cap=64, eos_id=1,
                 stream=stream.cuda_stream)
    res = []
    for rep in range(a.reps + 1):
        reqs = gen_requests(a.requests, shape, 1, 1, -1.0, 0, 64, 1, eos_id=1, p_range=(a.prompt, a.prompt),
                            first_id=1000 * rep)
        for r in reqs:
            eng.admit(r)
        p0 = eng.profile()
        eng.step(1)
        torch.cuda.synchronize()
        p1 = eng.profile()
        if rep:
            res.append(p1["prefill_ms"] - p0["prefill_ms"])
        eng.step(200)   # drain (cap 64 tokens)
        torch.cuda.synchronize()
    eng.close()
    P, qh, hd, L = a.prompt - 1, shape.n_heads, shape.head_dim, shape.n_layers
    attn_flop = a.requests * (L - 1) * qh * hd * 4.0 * P * (P + 1) / 2   # causal QK^T + PV
    ms = sorted(res)[len(res) // 2]
    print(json.dumps({"shape": a.shape, "prompt": a.prompt, "requests": a.requests,
                      "pf_umma": os.environ.get("SART_PF_UMMA", "1"), "prefill_ms_median": ms, "prefill_ms": res,
                      "prompt_tokens_per_s": a.requests * P / (ms / 1e3),
                      "attn_TFLOP": attn_flop / 1e12}))


if __name__ == "__main__":
    main()
