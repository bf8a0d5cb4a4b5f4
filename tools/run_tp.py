"""Row f4: the paper's 70B model with tensor parallelism, on the GPUs this process sees.

    python tools/run_tp.py [--tp 2] [--layers 80] [--windows 2] [--requests 8]

One process drives tp ranks (one ctx each, each on GPU rank % device_count, own stream, one
thread per rank); their receive buffers are connected with plain device pointers (peer access
between devices is enabled first when they differ).  On a one-GPU box all ranks share the
device: the run is a FUNCTIONAL check at full 70B size (141 GB of bf16 weights split over the
ranks, every O / down projection exchanged through the fused epilogue), not a TP performance
number -- the ranks then share one GPU's SMs and HBM.  Prints one JSON line: windows, tokens,
the ranks' agreement (identical tokens and records) and the timing.
"""
import argparse
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
# ranks sharing a device in one process: no lazy kernel loading (see tests/conftest.py)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--windows", type=int, default=2)
    ap.add_argument("--requests", type=int, default=8)
    ap.add_argument("--T", type=int, default=64)
    ap.add_argument("--cap", type=int, default=512)
    ap.add_argument("--num-blocks", type=int, default=600)
    a = ap.parse_args()
    import torch
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_requests
    shape = SHAPES["70B"] if a.layers == 80 else SHAPES["70B"].with_layers(a.layers)
    ndev = torch.cuda.device_count()
    devs = [r % ndev for r in range(a.tp)]
    t0 = time.time()
    engs = []
    for r in range(a.tp):
        engs.append(Engine(shape, "bf16", weight_seed=7, block_size=64, num_blocks=a.num_blocks, max_rows=128,
                           max_requests=64, max_prompt=1025, T=a.T, cap=a.cap, eos_id=1, temperature=1.0,
                           sampler_seed=3, device=devs[r], tp=(a.tp, r)))
    init_s = time.time() - t0
    ptrs = [e.tp_buffer()[0] for e in engs]
    for i, di in enumerate(devs):          # remote stores / atomics need peer access across devices
        for dj in set(devs):
            if dj != di:
                torch.cuda.set_device(di)
                try:
                    torch.cuda.cudart().cudaDeviceEnablePeerAccess(dj, 0)
                except Exception:
                    pass
    for e in engs:
        e.tp_connect(ptrs=ptrs)
    reqs = gen_requests(a.requests, shape, 8, 4, 0.5, 4, a.cap, a.T, eos_id=1, p_range=(64, 512))
    for e in engs:
        for q in reqs:
            e.admit(q)

    def all_ranks(fn):
        out = [None] * a.tp
        err = []

        def run(i):
            try:
                out[i] = fn(engs[i])
            except Exception as ex:   # noqa: BLE001
                err.append(ex)
        ts = [threading.Thread(target=run, args=(i,)) for i in range(a.tp)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        if err:
            raise err[0]
        return out

    all_ranks(lambda e: e.step(1))        # warm-up window (prefill + graph capture)
    torch.cuda.synchronize()
    s0 = [e.step(0) for e in engs]
    t = time.time()
    st = all_ranks(lambda e: e.step(a.windows))
    el = time.time() - t
    res = all_ranks(lambda e: e.collect())
    key = lambda rs: [(x["request_id"], x["answer_vote"], x["branch_len"], x["branch_state"], x["tokens"]) for x in rs]
    same = all(key(r) == key(res[0]) for r in res) and all(x == st[0] for x in st)
    steps = st[0]["steps"] - s0[0]["steps"]
    toks = st[0]["branch_tokens"] - s0[0]["branch_tokens"]
    print(json.dumps({"shape": shape.name, "tp": a.tp, "devices": devs, "init_s": init_s, "windows": a.windows,
                      "decode_steps": steps, "branch_tokens": toks, "wall_s": el,
                      "ms_per_decode_step": 1e3 * el / max(1, steps), "branch_tokens_per_s": toks / el,
                      "ranks_identical": same, "finalized": len(res[0]),
                      "note": "functional TP run; with all ranks on one GPU this is not a TP performance number"}),
          flush=True)
    for e in engs:
        e.close()


if __name__ == "__main__":
    main()
