"""In-graph marginal cost of each decode-step kernel class on the C2 bench workload.

    python tools/ablate_c2.py [--warm 3] [--windows 2] [--masks 0,1,2,...]

For each SART_ABLATE bit mask (sart_api.cu: 1 RMSNorm, 2 QKV, 4 attention, 8 attention merge,
16 O-proj, 32 gate/up, 64 down, 128 LM head, 256 sampler) a fresh process runs the bench's
C2 steady state (1.5B, 64 concurrent requests, N=8, T=400, CUDA-graph windows), warms up and
times whole windows with CUDA events.  The skipped kernels' results are garbage (rows still
terminate at their scripted lengths); only the time difference to mask 0 is meaningful: it
is what that kernel class costs inside the real graph, PDL overlap included, which a
serialised ncu launch list cannot show.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NAMES = {0: "baseline", 1: "rmsnorm", 2: "qkv", 4: "attention", 8: "attn_merge", 16: "o_proj", 32: "gate_up",
         64: "down", 128: "lm_head", 256: "sampler"}


def child(warm, windows):
    sys.path.insert(0, ROOT)
    import torch
    import bench
    from synth import SHAPES
    cfg = dict(bench.C2)
    shape = SHAPES["1.5B"]
    stream = torch.cuda.current_stream()
    eng = bench.make_engine(shape, cfg, 0, 0, stream, 0)
    for r in bench.make_requests(0, 1, 0, cfg["concurrent"] + 24 * (warm + windows), shape, cfg):
        eng.admit(r)
    eng.step(warm)
    torch.cuda.synchronize()
    s0 = eng.step(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.step(windows)
    e1.record(stream)
    torch.cuda.synchronize()
    s1 = eng.step(0)
    steps = s1["steps"] - s0["steps"]
    print(json.dumps({"ms": e0.elapsed_time(e1), "steps": steps, "ms_per_step": e0.elapsed_time(e1) / steps,
                      "rows_avg": (s1["branch_tokens"] - s0["branch_tokens"]) / max(1, steps)}), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--windows", type=int, default=2)
    ap.add_argument("--masks", default="0,1,2,4,8,16,32,64,128,256,0")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a.warm, a.windows)
        return
    base = None
    for m in [int(x) for x in a.masks.split(",")]:
        env = dict(os.environ, SART_ABLATE=str(m))
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", "--warm", str(a.warm),
                              "--windows", str(a.windows)], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(json.dumps({"mask": m, "error": out.stderr[-2000:]}), flush=True)
            continue
        r = json.loads(line[-1])
        if m == 0 and base is None:
            base = r["ms_per_step"]
        r.update(mask=m, skipped=NAMES.get(m, str(m)),
                 saved_ms_per_step=(base - r["ms_per_step"]) if base is not None else None)
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
