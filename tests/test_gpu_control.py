"""PP2: branch control on the GPU is bit-exact with the oracle replay.

Scripted workloads (forced EOS steps, scripted rewards and labels) make every control
decision a function of the script, so the oracle's Algorithm 1 engine (oracle/engine.py)
and the CUDA path (boundary/admission kernels through the C-ABI) must agree on every
integer after every window: row order, per-row steps, block tables, the free stack
(contents and order), commitment, meta[i] (phase, threshold bits, caps, counters, prefix
blocks), and the finalized records (votes, max-reward choice, branch states, lengths).
"""
import numpy as np
import pytest

from gpu_common import (compare_results, first_diff, gpu_engine, norm_gpu_state, norm_oracle_snapshot,
                        oracle_engine)
from synth import SHAPES, gen_requests, gen_weights

pytestmark = pytest.mark.gpu


def run_pair(shape, reqs, bs, nb, T, cap, B, select=0, windows=100000, check_every=1, es=False, prefill_chunk=0):
    g = gpu_engine(shape, "bf16", None, block_size=bs, num_blocks=nb, max_rows=B, max_requests=64, max_prompt=2048,
                   T=T, cap=cap, eos_id=1, select_mode=select, weight_seed=3, es_every_step=es,
                   prefill_chunk=prefill_chunk)
    o = oracle_engine(bs, nb, T, cap, B=B, select=select, es=es, prefill_chunk=prefill_chunk)
    for r in reqs:
        g.admit(r)
        o.admit(r)
    w = 0
    while w < windows:
        gs = g.step(1)
        o.step(1)
        w += 1
        if w % check_every == 0 or gs["live_rows"] == 0:
            a = norm_oracle_snapshot(o.snapshot())
            b = norm_gpu_state(g.state())
            d = first_diff(a, b)
            assert d is None, f"window {w}: first diverging field {d[0]}\n oracle={d[1]}\n gpu   ={d[2]}"
            assert gs["branch_tokens"] == o.branch_tokens and gs["steps"] == o.steps
        if gs["live_rows"] == 0 and gs["queued_requests"] == 0 and gs["queued_branches"] == 0:
            break
    gres, ores = g.collect(), o.collect()
    compare_results(gres, ores, {r.request_id: r.N for r in reqs})
    g.close()
    return gres


def test_trace_A_on_gpu():
    from tests_traces import trace_A_request
    shape = SHAPES["tiny"]
    res = run_pair(shape, [trace_A_request()], bs=16, nb=4096, T=16, cap=64, B=1 << 20)
    assert res[0]["num_pruned"] == 3 and res[0]["finalize_reason"] == 1


def test_trace_B_on_gpu():
    from tests_traces import trace_B_request
    shape = SHAPES["tiny"]
    run_pair(shape, [trace_B_request()], bs=16, nb=17, T=16, cap=64, B=1 << 20)


@pytest.mark.parametrize("seed", range(10))
def test_random_scripted_workloads(seed):
    rng = np.random.default_rng(100 + seed)
    shape = SHAPES["tiny"]
    bs = int(rng.choice([16, 64]))
    T = int(rng.choice([1, 4, 16]))
    cap = int(rng.integers(8, 160))
    N = int(rng.integers(1, 9))
    M = int(rng.integers(1, N + 1))
    reqs = gen_requests(int(rng.integers(2, 7)), shape, N, M, 0.5 if rng.random() < 0.7 else -1.0,
                        int(rng.integers(0, N)), cap, T, eos_id=1, p_range=(1, 150), length="uniform",
                        len_range=(1, cap), root_seed=seed)
    need = max(-(-(len(r.prompt) - 1) // bs) for r in reqs) + -(-cap // bs)
    nb = int(need + rng.integers(0, 3 * need))
    B = int(rng.integers(1, 3 * N + 1)) if rng.random() < 0.5 else 1024
    run_pair(shape, reqs, bs, nb, T, cap, B, select=int(rng.integers(0, 2)))


def test_paper_defaults_many_requests():
    """N=8, M=N/2, alpha=0.5, beta=N/2, a pool that forces queuing."""
    shape = SHAPES["tiny"]
    cap, T, bs = 96, 16, 16
    reqs = gen_requests(12, shape, 8, 4, 0.5, 4, cap, T, eos_id=1, p_range=(20, 120), root_seed=11)
    run_pair(shape, reqs, bs, nb=3 * (8 * 6 + 8), T=T, cap=cap, B=40, check_every=1)


def _mixed_requests(rng, shape, n, cap, T, first_id, root_seed):
    """n requests with independently drawn N, M, alpha, beta and prompt length (one engine
    serves them all; T, cap and bs are per-engine)."""
    from synth import Request, gen_prompt, gen_script
    reqs = []
    for i in range(n):
        rid = first_id + i
        N = int(rng.integers(1, 33))
        M = int(rng.integers(1, N + 1))
        alpha = float(np.float32(rng.choice([-1.0, 0.25, 0.5, 0.75])))
        beta = int(rng.integers(-1, N)) if N > 1 else 0
        sc = gen_script(rid, N, cap, T, "uniform", (1, cap), root_seed)
        reqs.append(Request(rid, gen_prompt(rid, shape.vocab, 1, 1, 200, root_seed), N, M, alpha, beta, sc))
    return reqs


@pytest.mark.parametrize("bs,T", [(16, 1), (16, 4), (64, 16), (64, 5), (16, 16), (64, 1)])
def test_many_mixed_requests_tight_pool(bs, T):
    """PP2 randomized coverage at volume: 150 requests per engine (900 over the parameter
    grid) with N up to 32, random M, alpha (incl. disabled), beta (incl. -1 -> N/2), a pool
    and row limit that force commitment stalls and queuing; every window bit-exact."""
    rng = np.random.default_rng(1000 * bs + T)
    shape = SHAPES["tiny"]
    cap = int(rng.integers(16, 120))
    reqs = _mixed_requests(rng, shape, 150, cap, T, 0, 7 + T)
    need = max(-(-(len(r.prompt) - 1) // bs) for r in reqs) + -(-cap // bs)
    nb = int(need * 6)
    run_pair(shape, reqs, bs, nb, T, cap, B=int(rng.integers(8, 64)))


@pytest.mark.parametrize("policy", ["vanilla", "self_consist", "sart_noprune", "sart"])
def test_policy_presets_match_oracle(policy):
    """NEXT row f3: the comparison policies (tools/policies.py) on the same engine are
    bit-exact with the oracle; Vanilla finalizes every request with its single branch and
    Self-Consistency completes all N branches."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from tools.policies import POLICIES
    from synth import Request, Script
    p = POLICIES[policy]
    shape = SHAPES["tiny"]
    cap, T, bs = 96, 16, 16
    reqs = gen_requests(10, shape, 8, p["M"], p["alpha"], p["beta"], cap, T, eos_id=1, p_range=(20, 120),
                        root_seed=21)
    if p["N"] < 8:
        reqs = [Request(r.request_id, r.prompt, p["N"], p["M"], p["alpha"], p["beta"],
                        Script(r.script.forced_len[:p["N"]], r.script.scores[:p["N"]],
                               r.script.final_score[:p["N"]], r.script.answer[:p["N"]])) for r in reqs]
    res = run_pair(shape, reqs, bs, nb=400, T=T, cap=cap, B=48)
    if policy == "vanilla":
        assert all(r["num_completed"] == 1 and r["num_pruned"] == 0 for r in res)
    if policy == "self_consist":
        assert all(r["num_completed"] == 8 and r["num_early_stopped"] == 0 for r in res)
    if policy == "sart_noprune":
        assert all(r["num_pruned"] == 0 and r["num_completed"] >= 2 for r in res)


def test_more_than_1024_rows():
    """B = 1500 rows resident at once (47 requests x N = 32): the window plan (k_attn_plan) keeps
    its per-row scratch in global memory, so batches above 1024 rows are exact too (ADVICE r1:
    a fixed __shared__ int[1024] used to overflow); control bit-exact with the oracle."""
    shape = SHAPES["tiny"]
    cap, T, bs = 32, 16, 16
    reqs = gen_requests(47, shape, 32, 16, 0.5, 16, cap, T, eos_id=1, p_range=(2, 60), length="uniform",
                        len_range=(1, cap), root_seed=31)
    res = run_pair(shape, reqs, bs, nb=4096, T=T, cap=cap, B=1500, check_every=1)
    assert len(res) == 47


def test_es_every_step_trace_B_on_gpu():
    """Reading R43 on the device (k_step_begin stops the rows, k_boundary early-stops them):
    trace B under es_every_step, bit-exact with the oracle every window."""
    from tests_traces import trace_B_request
    res = run_pair(SHAPES["tiny"], [trace_B_request()], bs=16, nb=17, T=16, cap=64, B=1 << 20, es=True)
    assert res[0]["branch_len"][:4] == [25, 10, 25, 25] and res[0]["window_final"] == 1


@pytest.mark.parametrize("seed", range(6))
def test_es_every_step_random_workloads(seed):
    """es_every_step with pruning on, mixed N / M / alpha / beta, tight pools: bit-exact."""
    rng = np.random.default_rng(500 + seed)
    shape = SHAPES["tiny"]
    bs = int(rng.choice([16, 64]))
    T = int(rng.choice([4, 16, 40]))
    cap = int(rng.integers(16, 120))
    reqs = _mixed_requests(rng, shape, 40, cap, T, 0, 70 + seed)
    need = max(-(-(len(r.prompt) - 1) // bs) for r in reqs) + -(-cap // bs)
    run_pair(shape, reqs, bs, int(need * 5), T, cap, B=int(rng.integers(8, 96)), es=True)


@pytest.mark.parametrize("seed", range(6))
def test_interleaved_prefill_random_workloads(seed):
    """Reading R44 (row f1): prefill chunks interleaved with decode steps -- rows of a request
    prefilled in the window start at the step its last chunk precedes.  Chunks of 8-48 tokens
    over prompts of up to 150 tokens spread a fill's prefill over many steps; mixed N / M /
    alpha / beta, tight pools, es_every_step on half the seeds: bit-exact every window."""
    rng = np.random.default_rng(900 + seed)
    shape = SHAPES["tiny"]
    bs = int(rng.choice([16, 64]))
    T = int(rng.choice([4, 16, 40]))
    cap = int(rng.integers(16, 100))
    reqs = _mixed_requests(rng, shape, 30, cap, T, 0, 90 + seed)
    need = max(-(-(len(r.prompt) - 1) // bs) for r in reqs) + -(-cap // bs)
    run_pair(shape, reqs, bs, int(need * 5), T, cap, B=int(rng.integers(8, 96)), es=bool(seed % 2),
             prefill_chunk=int(rng.choice([8, 16, 48])))
