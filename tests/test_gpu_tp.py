"""Row f4: tensor parallelism with the all-reduce fused into the O / down
GEMM epilogues, checked on ONE GPU.

Every gpurun call and the round-end tests have one B200, so the ranks of a TP group run on the
same device here: two ctx in one process (each with its own stream, driven by two threads, the
receive buffers exchanged as plain device pointers), or two processes exchanging CUDA IPC
handles -- the same peer-store / arrival-counter protocol the kernels use over NVLink.  What is
checked is what the sharding must preserve:
  * the model: teacher-forced logits, PRM scores and each rank's attention heads against the
    fp64 oracle of the FULL model (2e-2, bf16), at the small test shape and the 7B / 70B
    attention and FFN geometries;
  * replication: every rank computes bit-identical logits and tokens, so the replicated
    branch control stays identical -- scripted workloads are bit-exact with the oracle engine
    on every rank.
Performance of TP needs a multi-GPU box and is not measured here.
"""
import threading

import numpy as np
import pytest

from gpu_common import compare_results, first_diff, gpu_engine, norm_gpu_state, norm_oracle_snapshot, oracle_engine, rel_err_rows
from oracle.model import Model
from synth import SHAPES, Request, gen_prompt, gen_requests, gen_weights
from paper_2505_13326_b200 import DBG_ATTN, DBG_LOGITS, DBG_ROWIDS, DBG_SCORES

pytestmark = pytest.mark.gpu
EOS = 1


def tp_group(shape, weights, tp, **kw):
    engines = [gpu_engine(shape, "bf16", weights, tp=(tp, r), **kw) for r in range(tp)]
    ptrs = [e.tp_buffer()[0] for e in engines]
    for e in engines:
        e.tp_connect(ptrs=ptrs)
    return engines


def tp_call(engines, fn):
    """fn(engine) on every rank concurrently (the ranks' kernels wait for each other)."""
    out, err = [None] * len(engines), []

    def run(i):
        try:
            out[i] = fn(engines[i])
        except Exception as e:   # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(engines))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


def _slice(name, layers=1, vocab=4096):
    import dataclasses
    sh = SHAPES[name].with_layers(layers)
    return dataclasses.replace(sh, name=f"{name}-L{layers}-V{vocab}", vocab=vocab)


def teacher_forced_tp(shape, tp, prompts, N, steps, T, bs=16, std=0.02, seed=0, tol=2e-2):
    weights = gen_weights(shape, "bf16", std=std, root_seed=seed)
    model = Model(shape, weights)
    rng = np.random.default_rng(seed)
    eng = tp_group(shape, weights, tp, block_size=bs, num_blocks=1024, max_rows=64, max_requests=8,
                   max_prompt=max(len(p) for p in prompts) + 1, T=T, cap=steps, eos_id=EOS,
                   enable_forced_tokens=True, debug_capture=True)
    forced = {rid: rng.integers(2, shape.vocab, size=(N, steps)).astype(np.int32) for rid in range(len(prompts))}
    for e in eng:
        for rid, p in enumerate(prompts):
            e.admit(Request(rid, p, N, N, -1.0, 0, None), forced_tokens=forced[rid])
    layer = shape.n_layers - 1
    hq = shape.n_heads // tp * shape.head_dim
    worst = dict(logits=0.0, attn=0.0, prm=0.0)
    refs = {}
    for rid, p in enumerate(prompts):
        pre = model.prefill(p)
        for b in range(N):
            suf = [{"k": [], "v": []} for _ in range(shape.n_layers)]
            out = []
            for s in range(1, steps + 1):
                tok = p[-1] if s == 1 else forced[rid][b, s - 2]
                dbg = {}
                z, lg = model.decode(np.array([tok]), np.array([len(p) - 2 + s]), [pre], [suf], debug=dbg)
                out.append((lg[0], dbg["o"][layer][0], float(model.prm_score(z)[0])))
            refs[(rid, b)] = out
    for w in range(steps // T):
        tp_call(eng, lambda e: e.step(1))
        lgs = [e.debug_fetch(DBG_LOGITS) for e in eng]
        ats = [e.debug_fetch(DBG_ATTN, layer) for e in eng]
        scs = [e.debug_fetch(DBG_SCORES) for e in eng]
        ids = eng[0].debug_fetch(DBG_ROWIDS)
        for r in range(1, tp):   # replicated residual stream: bit-identical on every rank
            assert np.array_equal(lgs[r], lgs[0]) and np.array_equal(scs[r], scs[0])
            assert np.array_equal(eng[r].debug_fetch(DBG_ROWIDS), ids)
        s = (w + 1) * T
        for i, key in enumerate(ids):
            rid, b = int(key) >> 8, int(key) & 0xFF
            lg, o, prm = refs[(rid, b)][s - 1]
            e = rel_err_rows(lgs[0][i], lg)[0]
            worst["logits"] = max(worst["logits"], e)
            worst["prm"] = max(worst["prm"], abs(float(scs[0][i]) - prm))
            for r in range(tp):      # rank r holds q heads [r qh/tp, (r+1) qh/tp)
                worst["attn"] = max(worst["attn"], rel_err_rows(ats[r][i], o[r * hq:(r + 1) * hq])[0])
            assert e <= tol, (rid, b, s, e)
    res = tp_call(eng, lambda e: e.collect())
    for r in range(1, tp):
        assert [x["tokens"] for x in res[r]] == [x["tokens"] for x in res[0]]
    for e in eng:
        e.close()
    assert worst["attn"] <= tol and worst["prm"] <= tol, worst
    return worst


def test_tp2_small_teacher_forced():
    shape = SHAPES["small"]           # 8 q / 2 kv heads -> 4 / 1 per rank, F 1024 -> 512
    prompts = [gen_prompt(41, shape.vocab, EOS, 33, 33), gen_prompt(42, shape.vocab, EOS, 90, 90)]
    w = teacher_forced_tp(shape, 2, prompts, N=4, steps=48, T=8)
    print("TP=2 small worst", w)


@pytest.mark.parametrize("name", ["7B", pytest.param("70B", marks=pytest.mark.gpu_long)])
def test_tp2_geometry_teacher_forced(name):
    """7B (28/4 heads -> 14/2 per rank, F 18944 -> 9472) and the paper's 70B (64/8 ->
    32/4, d 8192, F 28672 -> 14336): one layer, small vocab."""
    shape = _slice(name)
    prompts = [gen_prompt(43, shape.vocab, EOS, 70, 70)]
    # reading R39: the bf16 bound is stated at the O1 logit scale; at d = 8192 the q.k logits of
    # std-0.02 weights are ~2.3x C2's and the attention output error of ANY bf16 path sits at
    # the bound (TP = 1 on the same rows: 1.8e-2, tools/check_70b_geometry.py) -- the 70B
    # geometry runs at std 0.01, where TP = 1 gives 0.44e-2
    std = 0.01 if shape.d_model >= 8192 else 0.02
    w = teacher_forced_tp(shape, 2, prompts, N=3, steps=16, T=8, bs=64, std=std)
    print(f"TP=2 {name}-L1 worst", w)


def test_tp4_small_teacher_forced():
    import dataclasses
    shape = dataclasses.replace(SHAPES["small"], name="small-kv4", n_kv_heads=4, d_ff=2048)   # 8/4 -> 2/1, F 512
    prompts = [gen_prompt(44, shape.vocab, EOS, 40, 40)]
    w = teacher_forced_tp(shape, 4, prompts, N=2, steps=16, T=4)
    print("TP=4 small worst", w)


def test_tp2_scripted_control_bit_exact():
    """The replicated control on a TP group: every rank's state equals the oracle engine's
    after every window, and the records match."""
    shape = SHAPES["small"]
    bs, T, cap, nb = 16, 8, 64, 600
    reqs = gen_requests(12, shape, 8, 4, 0.5, 4, cap, T, eos_id=EOS, p_range=(5, 60), length="uniform",
                        len_range=(1, cap), root_seed=9)
    eng = tp_group(shape, None, 2, block_size=bs, num_blocks=nb, max_rows=40, max_requests=16, max_prompt=64,
                   T=T, cap=cap, eos_id=EOS, weight_seed=4)
    o = oracle_engine(bs, nb, T, cap, B=40)
    for r in reqs:
        for e in eng:
            e.admit(r)
        o.admit(r)
    while True:
        st = tp_call(eng, lambda e: e.step(1))
        o.step(1)
        a = norm_oracle_snapshot(o.snapshot())
        for e in eng:
            d = first_diff(a, norm_gpu_state(e.state()))
            assert d is None, d
        if st[0]["live_rows"] == 0 and st[0]["queued_requests"] == 0 and st[0]["queued_branches"] == 0:
            break
    res = tp_call(eng, lambda e: e.collect())
    ores = o.collect()
    for r in res:
        compare_results(r, ores, {q.request_id: q.N for q in reqs})
    for e in eng:
        e.close()


def _ipc_worker(rank, port, q):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from gpu_common import gpu_engine as ge
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    shape = SHAPES["small"]
    weights = gen_weights(shape, "bf16", std=0.02, root_seed=3)
    e = ge(shape, "bf16", weights, tp=(2, rank), block_size=16, num_blocks=512, max_rows=16, max_requests=4,
           max_prompt=64, T=8, cap=16, eos_id=EOS, enable_forced_tokens=True, debug_capture=True)
    _, h = e.tp_buffer()
    hs = [None, None]
    dist.all_gather_object(hs, h)             # the IPC handles travel over the host group
    e.tp_connect(handles=hs)
    ft = np.random.default_rng(5).integers(2, shape.vocab, size=(2, 16)).astype(np.int32)
    e.admit(Request(0, gen_prompt(45, shape.vocab, EOS, 30, 30), 2, 2, -1.0, 0, None), forced_tokens=ft)
    lgs = []
    for _ in range(2):
        e.step(1)
        lgs.append(e.debug_fetch(DBG_LOGITS))
    e.close()
    q.put((rank, np.stack(lgs)))
    dist.barrier()
    dist.destroy_process_group()


def test_tp2_two_processes_ipc():
    """One process per rank, receive buffers exchanged as CUDA IPC handles (the multi-GPU
    path's plumbing): both ranks end with identical logits, equal to the in-process group's and
    within north_star's 2e-2 of the fp64 oracle of the full model.  (The two processes
    time-share ONE GPU here.  This is the test that exposed the init-ordering bug fixed in
    dalloc: a zeroing memset on the legacy stream, executed late, wiped state -- 4-6 of 16
    runs gave one of two fixed wrong answers before the fix, 0 of 10 after;
    profiles/r2_tp_ipc_flake.txt.)"""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got[0], got[1])
    shape = SHAPES["small"]
    weights = gen_weights(shape, "bf16", std=0.02, root_seed=3)
    eng = tp_group(shape, weights, 2, block_size=16, num_blocks=512, max_rows=16, max_requests=4, max_prompt=64,
                   T=8, cap=16, eos_id=EOS, enable_forced_tokens=True, debug_capture=True)
    ft = np.random.default_rng(5).integers(2, shape.vocab, size=(2, 16)).astype(np.int32)
    for e in eng:
        e.admit(Request(0, gen_prompt(45, shape.vocab, EOS, 30, 30), 2, 2, -1.0, 0, None), forced_tokens=ft)
    ref = []
    for _ in range(2):
        tp_call(eng, lambda e: e.step(1))
        ref.append(eng[0].debug_fetch(DBG_LOGITS))
    for e in eng:
        e.close()
    from oracle.model import Model
    model = Model(shape, weights)
    prompt = gen_prompt(45, shape.vocab, EOS, 30, 30)
    pre = model.prefill(prompt)
    worst = 0.0
    for b in range(2):
        suf = [{"k": [], "v": []} for _ in range(shape.n_layers)]
        for s in range(1, 17):
            tok = prompt[-1] if s == 1 else ft[b, s - 2]
            _, lg = model.decode(np.array([tok]), np.array([len(prompt) - 2 + s]), [pre], [suf])
            if s % 8 == 0:
                w = s // 8 - 1
                for src in (got[0], np.stack(ref)):
                    worst = max(worst, rel_err_rows(src[w][b], lg[0])[0])   # rows in admission order
    same = bool(np.array_equal(np.stack(ref), got[0]))
    print(f"TP=2 IPC: ranks identical, equal to the in-process group: {same}, worst vs oracle {worst:.3e}, "
          f"IPC vs in-process max {np.max(np.abs(np.stack(ref) - got[0])):.3e}")
    assert worst <= 2e-2
    assert same
