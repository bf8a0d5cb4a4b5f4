"""Row f4 on CPU: the tensor-parallel partitioning math, world size 2 over gloo.

The library decides which part of every tensor a TP rank holds (sart_debug_tp_segments, the
same code sart_init uses to cut its shard out of a full host blob).  Here each of two gloo
ranks builds its shard of a full random model from those segments, runs one decode step of
the decoder on its own q / kv heads and FFN rows in fp64 NumPy, and all-reduces the O-projection
and down-projection outputs (the exchange the GEMM epilogues do over NVLink) -- the logits
must equal the unsharded fp64 oracle's (oracle/model.py) to 1e-10, and every element of every
tensor must be held by exactly the rank the Megatron split assigns (heads / FFN rows).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth import SHAPES, gen_prompt, gen_weights, weight_names


def shard(shape, weights, tp, rank):
    from paper_2505_13326_b200.sart import debug_tp_segments
    out = {}
    for t, name in enumerate(weight_names(shape)):
        full = np.ascontiguousarray(weights[name], np.float64).ravel()
        segs = debug_tp_segments(shape, tp, rank, t)
        n = int(sum(s[1] for s in segs))
        loc = np.empty(n)
        for loff, cnt, cl, cf, c0, goff in segs:
            i = np.arange(cnt)
            loc[loff:loff + cnt] = full[goff + (i // cl) * cf + c0 + i % cl]
        out[name] = loc
    return out


def rank_decode(shape, w, tp, prefix_kv, toks, pos, rank):
    """One decode step of this rank's shard (heads [rank*qh/tp, ...), FFN rows [rank*F/tp, ...));
    the residual updates are all-reduced over the group."""
    from oracle.model import rmsnorm, rope, attention, silu
    d, hd, L = shape.d_model, shape.head_dim, shape.n_layers
    qr, kr, fr = shape.n_heads // tp, shape.n_kv_heads // tp, shape.d_ff // tp
    g = qr // kr
    h = w["embed"].reshape(shape.vocab, d)[toks]
    for l in range(L):
        a = rmsnorm(h, w[f"l{l}.attn_norm"], shape.rms_eps)
        y = a @ w[f"l{l}.wqkv"].reshape(-1, d).T + w[f"l{l}.bqkv"]
        q = y[:, : qr * hd].reshape(-1, qr, hd)
        k = y[:, qr * hd:(qr + kr) * hd].reshape(-1, kr, hd)
        v = y[:, (qr + kr) * hd:].reshape(-1, kr, hd)
        o = np.zeros((len(toks), qr, hd))
        for r in range(len(toks)):
            qq = rope(q[r], pos[r], shape.rope_theta)
            kk = rope(k[r], pos[r], shape.rope_theta)
            K = np.concatenate([prefix_kv[l]["k"][:, rank * kr:(rank + 1) * kr], kk[None]], 0)
            V = np.concatenate([prefix_kv[l]["v"][:, rank * kr:(rank + 1) * kr], v[r][None]], 0)
            for i in range(qr):
                o[r, i] = attention(qq[i], K[:, i // g], V[:, i // g])
        part = o.reshape(len(toks), -1) @ w[f"l{l}.wo"].reshape(d, qr * hd).T
        t = torch.from_numpy(part.copy())
        dist.all_reduce(t)                         # the O-projection exchange
        h = h + t.numpy()
        m = rmsnorm(h, w[f"l{l}.mlp_norm"], shape.rms_eps)
        gate = m @ w[f"l{l}.wgate"].reshape(fr, d).T
        up = m @ w[f"l{l}.wup"].reshape(fr, d).T
        part = (silu(gate) * up) @ w[f"l{l}.wdown"].reshape(d, fr).T
        t = torch.from_numpy(part.copy())
        dist.all_reduce(t)                         # the down-projection exchange
        h = h + t.numpy()
    z = rmsnorm(h, w["final_norm"], shape.rms_eps)
    return z @ w["lm_head"].reshape(shape.vocab, d).T


def _worker(rank, port, tp, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=tp)
    import dataclasses
    from oracle.model import Model
    shape = SHAPES["small"] if tp == 2 else dataclasses.replace(SHAPES["small"], name="small-kv4", n_kv_heads=4,
                                                                d_ff=2048)
    weights = gen_weights(shape, "fp32", std=0.05, root_seed=12)
    w = shard(shape, weights, tp, rank)
    model = Model(shape, weights)
    prompt = gen_prompt(3, shape.vocab, 1, 20, 20)
    pre = model.prefill(prompt)
    toks = np.array([prompt[-1], 7])
    pos = np.array([len(prompt) - 1, len(prompt) - 1])
    lg = rank_decode(shape, w, tp, pre, toks, pos, rank)
    suf = [[{"k": [], "v": []} for _ in range(shape.n_layers)] for _ in range(2)]
    _, ref = model.decode(toks, pos, [pre, pre], suf)
    q.put((rank, float(np.max(np.abs(lg - ref)) / np.max(np.abs(ref))), {k: v.size for k, v in w.items()}))
    dist.destroy_process_group()


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_shards_reproduce_the_full_decoder(tp):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    qq = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, port, tp, qq)) for r in range(tp)]
    for p in ps:
        p.start()
    got = [qq.get(timeout=300) for _ in range(tp)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, sizes in got:
        assert err < 1e-10, (rank, err)


def test_tp_segments_partition_every_tensor():
    """Every element of every sharded tensor is held by exactly one rank, at the position the
    Megatron split gives it (replicated tensors by every rank), enumerated exactly on shapes
    with the small test and the 7B / 70B head geometries (small d / F / V keep it fast)."""
    import dataclasses
    from paper_2505_13326_b200.sart import debug_tp_segments
    from synth import weight_shapes
    shapes = [SHAPES["small"],
              dataclasses.replace(SHAPES["7B"], name="7b-mini", n_layers=1, d_model=128, d_ff=1024, vocab=64),
              dataclasses.replace(SHAPES["70B"], name="70b-mini", n_layers=1, d_model=128, d_ff=2048, vocab=64)]
    for sh in shapes:
        for tp in (2, 4, 8):
            if sh.n_heads % tp or sh.n_kv_heads % tp or (sh.d_ff // tp) % 128 or sh.d_ff % tp:
                continue
            shp = weight_shapes(sh)
            for t, wn in enumerate(weight_names(sh)):
                n = int(np.prod(shp[wn]))
                count = np.zeros(n, np.int64)
                owner = np.full(n, -1, np.int64)
                for rank in range(tp):
                    for loff, cnt, cl, cf, c0, goff in debug_tp_segments(sh, tp, rank, t):
                        i = np.arange(cnt)
                        gi = goff + (i // cl) * cf + c0 + i % cl
                        assert gi.min() >= 0 and gi.max() < n
                        count[gi] += 1
                        owner[gi] = rank
                sharded = any(wn.endswith(x) for x in (".wqkv", ".bqkv", ".wo", ".wgate", ".wup", ".wdown"))
                assert np.all(count == (1 if sharded else tp)), (sh.name, tp, wn)
                if not sharded:
                    continue
                hd, qh, kvh = sh.head_dim, sh.n_heads, sh.n_kv_heads
                if wn.endswith((".wqkv", ".bqkv")):      # output rows: q heads, k heads, v heads
                    width = sh.d_model if wn.endswith(".wqkv") else 1
                    row = np.arange(n) // width
                    head = row // hd
                    want = np.where(head < qh, head // (qh // tp),
                                    np.where(head < qh + kvh, (head - qh) // (kvh // tp),
                                             (head - qh - kvh) // (kvh // tp)))
                elif wn.endswith(".wo"):                  # input columns = q head dims
                    want = (np.arange(n) % (qh * hd)) // hd // (qh // tp)
                elif wn.endswith((".wgate", ".wup")):     # output rows = FFN rows
                    want = (np.arange(n) // sh.d_model) // (sh.d_ff // tp)
                else:                                     # wdown: input columns = FFN rows
                    want = (np.arange(n) % sh.d_ff) // (sh.d_ff // tp)
                assert np.array_equal(owner, want), (sh.name, tp, wn)
