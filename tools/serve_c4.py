"""C4 (BASELINE.json configs[3]): Poisson-arrival serving on one GPU.

7B shape, N=8, M=2, aggressive pruning (alpha 0.8, beta 4), cap 8192, T=400, FCFS admission on
freed KV blocks (commitment, R34).  Requests are admitted when their (Poisson) arrival time
has passed on the host clock; windows run back to back; latencies come from the result
records: E2E = final - arrival, queuing = prefill start - arrival (R27), inference = E2E -
queuing.  Percentiles are nearest-rank.

    python tools/serve_c4.py --requests 120 --rate 1.0
    python tools/serve_c4.py --prm PRM-7B     # scores from a separate PRM-7B decoder (row f2)

Without --prm the pruning scores are the synthetic script's (DESIGN.md input recipe); with
--prm they come from the separate PRM model (random-init weights: the pruning decisions are
then arbitrary, but the serving cost -- a 7B forward over every branch's new tokens at each
boundary -- is the paper's).
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def nearest_rank(xs, p):
    s = sorted(xs)
    if not s:
        return None
    k = max(1, math.ceil(p / 100.0 * len(s)))
    return s[k - 1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=120)
    ap.add_argument("--rate", type=float, default=1.0)
    ap.add_argument("--shape", default="7B")
    ap.add_argument("--cap", type=int, default=8192)
    ap.add_argument("--T", type=int, default=400)
    ap.add_argument("--prm", default=None, help="separate PRM decoder shape (row f2), e.g. PRM-7B")
    a = ap.parse_args()
    import torch
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_arrivals, gen_requests
    shape = SHAPES[a.shape]
    prm = None
    if a.prm:   # the PRM reads the policy's tokens: give it the policy's vocab
        import dataclasses
        prm = dataclasses.replace(SHAPES[a.prm], vocab=shape.vocab)
    stream = torch.cuda.current_stream()
    eng = Engine(shape, "bf16", weight_seed=4, block_size=64, num_blocks=0, max_rows=1024, max_requests=512,
                 max_prompt=1025, T=a.T, cap=a.cap, eos_id=1, temperature=1.0, sampler_seed=9,
                 stream=stream.cuda_stream, prm_shape=prm, prm_weight_seed=12)
    reqs = gen_requests(a.requests, shape, 8, 2, 0.8, 4, a.cap, a.T, eos_id=1, p_range=(64, 1024))
    arr = gen_arrivals(a.requests, a.rate)            # ns offsets of a Poisson process
    t0 = time.monotonic_ns()
    nxt = 0
    results = []
    windows = 0
    while len(results) < a.requests:
        now = time.monotonic_ns() - t0
        while nxt < a.requests and arr[nxt] <= now:
            reqs[nxt].arrival_ns = t0 + int(arr[nxt])     # absolute, same clock as the engine
            eng.admit(reqs[nxt], use_script_scores=prm is None)
            nxt += 1
        st = eng.step(1)
        windows += 1
        results += eng.collect()
        if st["live_rows"] == 0 and st["queued_requests"] == 0 and st["queued_branches"] == 0 and nxt < a.requests:
            time.sleep(max(0.0, (arr[nxt] - (time.monotonic_ns() - t0)) / 1e9))
    wall = (time.monotonic_ns() - t0) / 1e9
    e2e = [(r["t_final_ns"] - r["t_arrival_ns"]) / 1e9 for r in results]
    que = [(r["t_prefill_ns"] - r["t_arrival_ns"]) / 1e9 for r in results]
    inf = [x - y for x, y in zip(e2e, que)]
    pct = lambda xs: {f"p{p}": nearest_rank(xs, p) for p in (50, 90, 97, 99)}
    st = eng.step(0)
    prof = eng.profile()
    out = {"config": "C4 (BJ configs[3]) single GPU", "shape": a.shape, "prm_model": a.prm,
           "prm_ms_per_boundary": prof["prm_ms"] / max(1, prof["prm_passes"]) if a.prm else None,
           "prm_share_of_wall": prof["prm_ms"] / 1e3 / wall if a.prm else None, "requests": a.requests,
           "rate_req_per_s": a.rate, "wall_s": wall, "requests_per_s": a.requests / wall,
           "branch_tokens_per_s": st["branch_tokens"] / wall, "windows": windows,
           "e2e_s": pct(e2e), "queuing_s": pct(que), "inference_s": pct(inf),
           "pruned_branches": sum(r["num_pruned"] for r in results),
           "early_stopped_branches": sum(r["num_early_stopped"] for r in results),
           "completed_branches": sum(r["num_completed"] for r in results),
           "discarded_branches": sum(r["num_discarded_queued"] for r in results)}
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
