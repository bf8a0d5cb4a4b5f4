"""Debug: the two-process CUDA-IPC TP group vs the fp64 oracle (prints per-window logits errors)."""
import os
import socket
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402


def ref_logits(shape, weights, prompt, ft, steps):
    from oracle.model import Model
    m = Model(shape, weights)
    pre = m.prefill(prompt)
    out = {}
    for b in range(2):
        suf = [{"k": [], "v": []} for _ in range(shape.n_layers)]
        for s in range(1, steps + 1):
            tok = prompt[-1] if s == 1 else ft[b, s - 2]
            _, lg = m.decode(np.array([tok]), np.array([len(prompt) - 2 + s]), [pre], [suf])
            out[(b, s)] = lg[0]
    return out


def worker(rank, port):
    import torch.distributed as dist
    from gpu_common import gpu_engine
    from synth import SHAPES, Request, gen_prompt, gen_weights
    from paper_2505_13326_b200 import DBG_LOGITS, DBG_ROWIDS
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    shape = SHAPES["small"]
    weights = gen_weights(shape, "bf16", std=0.02, root_seed=3)
    e = gpu_engine(shape, "bf16", weights, tp=(2, rank), block_size=16, num_blocks=512, max_rows=16, max_requests=4,
                   max_prompt=64, T=8, cap=16, eos_id=1, enable_forced_tokens=True, debug_capture=True)
    _, h = e.tp_buffer()
    hs = [None, None]
    dist.all_gather_object(hs, h)
    e.tp_connect(handles=hs)
    ft = np.random.default_rng(5).integers(2, shape.vocab, size=(2, 16)).astype(np.int32)
    prompt = gen_prompt(45, shape.vocab, 1, 30, 30)
    e.admit(Request(0, prompt, 2, 2, -1.0, 0, None), forced_tokens=ft)
    ref = ref_logits(shape, weights, prompt, ft, 16)
    errs = []
    for w in range(2):
        e.step(1)
        lg = e.debug_fetch(DBG_LOGITS)
        ids = e.debug_fetch(DBG_ROWIDS)
        for i, k in enumerate(ids):
            b = int(k) & 0xFF
            r = ref[(b, 8 * (w + 1))]
            errs.append(f"w{w}b{b} {np.max(np.abs(lg[i] - r)) / np.max(np.abs(r)):.3e}")
    print(f"rank {rank} rel err " + " ".join(errs), flush=True)
    e.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=worker, args=(r, port)) for r in range(2)]
    [p.start() for p in ps]
    [p.join() for p in ps]
