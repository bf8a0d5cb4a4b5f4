"""NEXT row f3: the paper's comparison policies on the same engine, plus the occupancy trace.

SURVEY §8(f) f3 / PAPER P:154-166 (Fig. 3), P:333-338 (baselines), P:384-391 (Fig. 6 ablation):
  vanilla        N=1, M=1, no pruning                      (SART with N=M=1 == Vanilla)
  self_consist   N=8, M=8, no pruning, majority vote        (Self-Consistency)
  sart_noprune   N=8, M=2, no pruning                       ("SART w/o pruning")
  sart           N=8, M=2, alpha=0.8, beta=4                (C4's aggressive threshold)
Every policy serves the same Poisson-arrival trace of scripted requests (DESIGN.md input
recipe: lognormal lengths, Beta(4,2) label correctness independent of length, rewards by
correctness) through the C-ABI on one GPU.  Reported per policy: E2E / queuing / inference
latency percentiles (nearest rank), requests/s, generated tokens per request, the
synthetic vote accuracy (answer label 0 = correct -- a property of the synthetic recipe, not
the paper's GPQA/GAOKAO accuracy, which needs trained weights) and the occupancy trace
(live rows / free and committed KV blocks per window, the analogue of Fig. 4).

    python tools/policies.py [--shape 1.5B] [--requests 64] [--rate 4] [--policies ...]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.serve_c4 import nearest_rank  # noqa: E402

POLICIES = {
    "vanilla": dict(N=1, M=1, alpha=-1.0, beta=0),
    "self_consist": dict(N=8, M=8, alpha=-1.0, beta=4),
    "sart_noprune": dict(N=8, M=2, alpha=-1.0, beta=4),
    "sart": dict(N=8, M=2, alpha=0.8, beta=4),
}


def run_policy(name, shape, a, engine_cls, gen_requests, gen_arrivals, stream):
    p = POLICIES[name]
    eng = engine_cls(shape, "bf16", weight_seed=4, block_size=64, num_blocks=a.num_blocks, max_rows=1024,
                     max_requests=512, max_prompt=1025, T=a.T, cap=a.cap, eos_id=1, temperature=1.0,
                     sampler_seed=9, stream=stream)
    # the same workload for every policy: request r's prompt and branch scripts come from
    # the same named streams, so branch b of request r is identical across policies
    reqs = gen_requests(a.requests, shape, 8, p["M"], p["alpha"], p["beta"], a.cap, a.T, eos_id=1,
                        p_range=(64, 1024))
    if p["N"] < 8:
        from synth import Request, Script
        cut = []
        for r in reqs:
            s = r.script
            sc = Script(s.forced_len[:p["N"]], s.scores[:p["N"]], s.final_score[:p["N"]], s.answer[:p["N"]])
            cut.append(Request(r.request_id, r.prompt, p["N"], p["M"], p["alpha"], p["beta"], sc))
        reqs = cut
    arr = gen_arrivals(a.requests, a.rate)
    t0 = time.monotonic_ns()
    nxt, results, trace = 0, [], []
    while len(results) < a.requests:
        now = time.monotonic_ns() - t0
        while nxt < a.requests and arr[nxt] <= now:
            reqs[nxt].arrival_ns = t0 + int(arr[nxt])
            eng.admit(reqs[nxt])
            nxt += 1
        st = eng.step(1)
        results += eng.collect()
        trace.append([round((time.monotonic_ns() - t0) / 1e9, 3), st["live_rows"], st["free_blocks"],
                      st["committed_blocks"], st["queued_requests"]])
        if st["live_rows"] == 0 and st["queued_requests"] == 0 and st["queued_branches"] == 0 and nxt < a.requests:
            time.sleep(max(0.0, (arr[nxt] - (time.monotonic_ns() - t0)) / 1e9))
    wall = (time.monotonic_ns() - t0) / 1e9
    st = eng.step(0)
    eng.close()
    e2e = [(r["t_final_ns"] - r["t_arrival_ns"]) / 1e9 for r in results]
    que = [(r["t_prefill_ns"] - r["t_arrival_ns"]) / 1e9 for r in results]
    inf = [x - y for x, y in zip(e2e, que)]
    pct = lambda xs: {f"p{q}": nearest_rank(xs, q) for q in (50, 90, 97, 99)}
    return {"policy": name, **p, "shape": shape.name, "requests": a.requests, "rate_req_per_s": a.rate,
            "wall_s": wall, "requests_per_s": a.requests / wall, "branch_tokens_per_s": st["branch_tokens"] / wall,
            "tokens_per_request": st["branch_tokens"] / a.requests,
            "vote_accuracy_synthetic": sum(r["answer_vote"] == 0 for r in results) / len(results),
            "e2e_s": pct(e2e), "queuing_s": pct(que), "inference_s": pct(inf),
            "completed": sum(r["num_completed"] for r in results), "pruned": sum(r["num_pruned"] for r in results),
            "early_stopped": sum(r["num_early_stopped"] for r in results),
            "occupancy_trace": {"columns": ["t_s", "live_rows", "free_blocks", "committed_blocks", "queued_requests"],
                                "rows": trace}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="1.5B")
    ap.add_argument("--requests", type=int, default=64)
    ap.add_argument("--rate", type=float, default=4.0)
    ap.add_argument("--cap", type=int, default=4096)
    ap.add_argument("--T", type=int, default=400)
    ap.add_argument("--num-blocks", type=int, default=0, help="0 = size the KV pool from free HBM")
    ap.add_argument("--policies", nargs="*", default=list(POLICIES))
    a = ap.parse_args()
    import torch
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_arrivals, gen_requests
    shape = SHAPES[a.shape]
    stream = torch.cuda.current_stream().cuda_stream
    for name in a.policies:
        print(json.dumps(run_policy(name, shape, a, Engine, gen_requests, gen_arrivals, stream)), flush=True)


if __name__ == "__main__":
    main()
