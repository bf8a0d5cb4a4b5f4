"""Row f1 (reading R44): what interleaving the prefill with decode does to resident rows.

    python tools/interleave_demo.py [--chunks 0,2048,512]

C2-like residents (1.5B, 48 requests x N = 8 decoding, cap 4096) when two long prompts (8192
tokens each) arrive: their prefill (16K tokens) either runs before the window's first decode
step (prefill_chunk = 0, Alg. 1 L7 inline) or in chunks interleaved with the window's decode
steps.  For the admission window (profile mode: eager launches, CUDA events per step) it prints
the time from the window's start to its first decode step and the longest single step -- the
stall the resident rows see -- and the window's total time.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(chunk, warm=2):
    import torch
    import bench
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_requests
    shape = SHAPES["1.5B"]
    cfg = dict(bench.C2)
    stream = torch.cuda.current_stream()
    eng = Engine(shape, "bf16", weight_seed=5, block_size=64, num_blocks=0, max_rows=512, max_requests=256,
                 max_prompt=8193, T=400, cap=4096, eos_id=1, temperature=1.0, sampler_seed=7,
                 stream=stream.cuda_stream, prefill_chunk=chunk)
    for r in bench.make_requests(0, 1, 0, 48, shape, cfg):
        eng.admit(r)
    eng.step(warm)
    late = gen_requests(2, shape, 8, 4, -1.0, 4, 4096, 400, eos_id=1, p_range=(8193, 8193), first_id=1 << 16)
    for r in late:
        eng.admit(r)
    torch.cuda.synchronize()
    eng.set_profile(True)
    eng.reset_profile()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    st = eng.step(1)
    e1.record(stream)
    torch.cuda.synchronize()
    p = eng.profile()
    eng.close()
    return {"prefill_chunk": chunk, "window_ms": e0.elapsed_time(e1), "first_step_ms": p["first_step_ms_max"],
            "max_step_ms": p["step_ms_max"], "live_rows": st["live_rows"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", default="0,2048,512")
    a = ap.parse_args()
    for c in [int(x) for x in a.chunks.split(",")]:
        print(json.dumps(run(c)), flush=True)


if __name__ == "__main__":
    main()
