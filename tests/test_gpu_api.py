"""C-ABI behaviour on the GPU: error codes and all-or-nothing validation (include/sart.h),
determinism (PP4: same seeds -> identical results, model mode with float reductions), the
counter export used by the multi-GPU all-gather, and result collection with small buffers."""
import ctypes as C

import numpy as np
import pytest

from gpu_common import gpu_engine
from synth import SHAPES, Request, Script, gen_prompt, gen_requests, gen_weights

pytestmark = pytest.mark.gpu
EOS = 1


def eng(**kw):
    shape = SHAPES["tiny"]
    base = dict(block_size=16, num_blocks=512, max_rows=64, max_requests=16, max_prompt=64, T=8, cap=32, eos_id=EOS)
    base.update(kw)
    return gpu_engine(shape, "bf16", None, weight_seed=5, **base)


def test_admit_validation_codes():
    from paper_2505_13326_b200.sart import SartError, SART_EINVAL, SART_EDUP, SART_ENOMEM
    g = eng()
    p = gen_prompt(0, 512, EOS, 5, 5)
    bad = [Request(0, p, 4, 5, 0.5, 1, None),            # M > N
           Request(0, p, 33, 2, 0.5, 1, None),           # N > 32
           Request(0, p, 4, 2, 0.5, 4, None),            # beta > N-1
           Request(0, p, 4, 2, 1.5, 1, None),            # alpha > 1
           Request(0, p, 4, 2, float("nan"), 1, None),   # alpha NaN
           Request(0, np.array([], np.int32), 4, 2, 0.5, 1, None)]
    for r in bad:
        with pytest.raises(SartError) as e:
            g.admit(r)
        assert e.value.code == SART_EINVAL
    half = Script(np.array([3, 3], np.int32), np.zeros((2, 2), np.float32), None, None)
    with pytest.raises(SartError) as e:     # scores without final_score: half-specified script
        g.admit(Request(1, p, 2, 1, 0.5, 0, half))
    assert e.value.code == SART_EINVAL
    g.admit(Request(7, p, 2, 1, 0.5, -1, None))          # beta = -1 -> N/2
    with pytest.raises(SartError) as e:
        g.admit(Request(7, p, 2, 1, 0.5, 0, None))
    assert e.value.code == SART_EDUP
    with pytest.raises(SartError) as e:                  # could never fit: prefix 4 blocks + row 2 > NB
        small = eng(num_blocks=4)
        small.admit(Request(9, gen_prompt(1, 512, EOS, 60, 60), 1, 1, 0.5, 0, None))
    assert e.value.code == SART_ENOMEM
    st = g.step(100)                                     # the valid request still runs to completion
    assert st["finalized_total"] == 1 and st["live_rows"] == 0
    g.close()


def test_init_validation_codes():
    from paper_2505_13326_b200.sart import SartError, SART_EINVAL, SART_ENOMEM
    import dataclasses
    bad_shape = dataclasses.replace(SHAPES["tiny"], head_dim=96)
    with pytest.raises(SartError) as e:
        gpu_engine(bad_shape, "bf16", None, num_blocks=64, max_prompt=64, T=8, cap=32)
    assert e.value.code == SART_EINVAL
    with pytest.raises(SartError) as e:
        eng(block_size=48)
    assert e.value.code == SART_EINVAL
    with pytest.raises(SartError) as e:
        eng(num_blocks=1)                                  # < ceil(cap / bs) = 2
    assert e.value.code == SART_ENOMEM
    # row f2: a separate PRM decoder with an unsupported head_dim / GQA ratio / FFN width
    for bad in (dict(head_dim=96), dict(n_kv_heads=4), dict(d_ff=1000)):
        with pytest.raises(SartError) as e:
            eng(prm_shape=dataclasses.replace(SHAPES["prm-tiny"], **bad))
        assert e.value.code == SART_EINVAL, bad
    with pytest.raises(ValueError):                        # the PRM reads the policy's vocab
        eng(prm_shape=dataclasses.replace(SHAPES["prm-tiny"], vocab=1024))


def run_model_mode(seed):
    shape = SHAPES["tiny"]
    w = gen_weights(shape, "bf16", std=0.08)
    w["lm_head"][EOS] *= 5.0
    g = gpu_engine(shape, "bf16", w, block_size=16, num_blocks=1024, max_rows=64, max_requests=16, max_prompt=64,
                   T=8, cap=40, eos_id=EOS, temperature=1.0, sampler_seed=seed)
    for rid in range(6):
        g.admit(Request(rid, gen_prompt(rid, shape.vocab, EOS, 8, 40), 6, 3, 0.4, 3, None))
    g.step(1000)
    res = g.collect()
    g.close()
    return res


def test_determinism_model_mode():
    """PP4: identical seeds give identical tokens, scores and decisions (fixed reduction orders)."""
    a, b = run_model_mode(11), run_model_mode(11)
    assert len(a) == len(b) == 6
    clock = ("t_arrival_ns", "t_prefill_ns", "t_final_ns")
    for x, y in zip(a, b):
        assert {k: v for k, v in x.items() if k not in clock} == {k: v for k, v in y.items() if k not in clock}
    c = run_model_mode(12)
    assert any(x["tokens"] != y["tokens"] for x, y in zip(a, c))     # the seed matters


def test_collect_partial_buffers_and_counters():
    import torch
    g = eng()
    reqs = gen_requests(5, SHAPES["tiny"], 3, 2, -1.0, 0, 32, 8, eos_id=EOS, p_range=(3, 20), length="uniform",
                        len_range=(1, 32), root_seed=3)
    for r in reqs:
        g.admit(r)
    g.step(1000)
    dev = torch.zeros(16, dtype=torch.int32, device="cuda")
    g.export_counters(dev.data_ptr())
    torch.cuda.synchronize()
    c = dev.cpu().tolist()
    assert c[0] == 0 and c[5] == 5 and c[3] == 512 and c[4] == 0    # live rows, finalized, free, committed
    from paper_2505_13326_b200.sart import SartResult, P32, SART_EFULL
    res = (SartResult * 2)()
    toks = np.zeros(1000, np.int32)
    n = C.c_int32()
    rc = g.lib.sart_collect(g.ctx, res, 2, C.byref(n), toks.ctypes.data_as(P32), 1000)
    assert rc == SART_EFULL and n.value == 2
    rest = g.collect()
    assert len(rest) == 3
    assert sorted([res[0].request_id, res[1].request_id] + [r["request_id"] for r in rest]) == [0, 1, 2, 3, 4]
    g.close()


def test_forced_token_out_of_range_rejected():
    """forced tokens become embedding indices -- out-of-range ids are EINVAL."""
    from paper_2505_13326_b200.sart import SartError, SART_EINVAL
    g = eng(enable_forced_tokens=True)
    p = gen_prompt(0, 512, EOS, 5, 5)
    ft = np.full((2, 32), 7, np.int32)
    ft[1, 5] = 512
    with pytest.raises(SartError) as e:
        g.admit(Request(0, p, 2, 1, -1.0, 0, None), forced_tokens=ft)
    assert e.value.code == SART_EINVAL
    ft[1, 5] = -1
    with pytest.raises(SartError) as e:
        g.admit(Request(0, p, 2, 1, -1.0, 0, None), forced_tokens=ft)
    assert e.value.code == SART_EINVAL
    ft[1, 5] = 511
    g.admit(Request(0, p, 2, 1, -1.0, 0, None), forced_tokens=ft)
    assert g.step(100)["finalized_total"] == 1


def test_dist_serve_with_cuda_engine_world1():
    """SURVEY §8(e) on the real engine: dist.serve drives sart_admit / sart_step / sart_collect
    and the C1 counter all-gather over NCCL (world size 1 on this one-GPU box); the result
    records then go through the C2 tensor gather.  Equal to running the engine directly."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2505_13326_b200 import dist as sdist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        shape = SHAPES["tiny"]
        reqs = gen_requests(9, shape, 4, 2, 0.5, 2, 32, 8, eos_id=EOS, p_range=(2, 40), length="uniform",
                            len_range=(1, 32), root_seed=17)
        arrivals = [reqs[0:3], [], reqs[3:7], reqs[7:9]]
        seen = []
        res = sdist.serve(eng(), arrivals, policy="least_loaded", on_window=lambda w, st, c: seen.append(c.clone()))
        assert all(c.is_cuda and c.shape == (1, 16) for c in seen)
        assert int(seen[-1][0, sdist.FINALIZED]) == 9
        recs = sdist.gather_result_records(res, "cuda:0")
        ref_eng = eng()
        for r in reqs:
            ref_eng.admit(r)
        ref_eng.step(1000)
        ref = {r["request_id"]: r for r in ref_eng.collect()}
        assert sorted(r["request_id"] for r in res) == sorted(ref)
        for r in res:
            o = ref[r["request_id"]]
            for k in ("answer_vote", "num_completed", "num_pruned", "num_early_stopped", "branch_len",
                      "branch_state"):
                assert r[k] == o[k], k
        assert recs.shape == (9, len(sdist.RECORD_FIELDS))
        assert sorted(recs[:, 0].tolist()) == sorted(ref)
    finally:
        dist.destroy_process_group()


def test_kv_pool_caller_owned():
    """SURVEY §8(b) kv_pool: a torch-allocated device buffer as the KV pool (filled with NaN to
    prove the engine zeroes it) gives exactly the results of the engine-owned pool."""
    import torch
    shape = SHAPES["tiny"]
    reqs = gen_requests(6, shape, 4, 2, 0.5, 2, 32, 8, eos_id=EOS, p_range=(2, 40), length="uniform",
                        len_range=(1, 32), root_seed=23)
    weights = gen_weights(shape, "bf16", std=0.08)
    ref = gpu_engine(shape, "bf16", weights, block_size=16, num_blocks=200, max_rows=64, max_requests=16,
                     max_prompt=64, T=8, cap=32, eos_id=EOS, sampler_seed=3)
    for r in reqs:
        ref.admit(r)
    ref.step(100)
    want = ref.collect()
    ref.close()
    blk = shape.n_layers * 2 * shape.n_kv_heads * 16 * shape.head_dim * 2      # bf16 bytes per block
    pool = torch.full((200 * blk // 2,), float("nan"), dtype=torch.bfloat16, device="cuda")
    g = gpu_engine(shape, "bf16", weights, block_size=16, num_blocks=0, max_rows=64, max_requests=16, max_prompt=64,
                   T=8, cap=32, eos_id=EOS, sampler_seed=3, kv_pool=(pool.data_ptr(), pool.numel() * 2))
    for r in reqs:
        g.admit(r)
    g.step(100)
    got = g.collect()
    g.close()
    keys = ("request_id", "answer_vote", "branch_len", "branch_state", "branch_score", "tokens")
    assert [{k: x[k] for k in keys} for x in got] == [{k: x[k] for k in keys} for x in want]
