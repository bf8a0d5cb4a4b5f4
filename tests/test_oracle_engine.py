"""Pins for oracle/engine.py (Algorithm 1, plus readings R2-R35).

* Hand traces A and B, derived by hand from Alg. 1 and the O8 allocator.
* SPEC worked examples S:271-273 (pruning, phase switch, early stop), S:280-282 (vote,
  max reward).
* Brute force: random scripts on tiny branch sets vs an independent, naive line-by-line
  transcription of Alg. 1 without an allocator (below), plus the predicates the paper fixes.
* Allocator invariants on random multi-request workloads with a tight pool.
* Vote: exhaustive over label vectors vs plurality computed another way.
* Degenerate policies: N=M=1, alpha=0, beta=0 is Vanilla; M=N without pruning is
  Self-Consistency.
"""
import collections
import itertools

import numpy as np
import pytest

from oracle.engine import (COMPLETED_CAP, COMPLETED_EOS, DISCARDED, EARLY_STOPPED, EXPLOIT,
                           EXPLORE, PRUNED, Engine, EngineConfig, ScriptedSource)
from synth import Request, Script, gen_requests, SHAPES

COMPLETED = (COMPLETED_EOS, COMPLETED_CAP)


def mk_req(rid, lengths, scores, finals=None, answers=None, M=2, alpha=0.5, beta=2, P=3):
    N = len(lengths)
    sc = np.asarray(scores, np.float32)
    fin = np.asarray(finals if finals is not None else [0.5] * N, np.float32)
    ans = np.asarray(answers if answers is not None else [0] * N, np.int32)
    return Request(rid, np.arange(2, 2 + P, dtype=np.int32), N, M, float(np.float32(alpha)), beta,
                   Script(np.asarray(lengths, np.int32), sc, fin, ans))


def engine(T=16, cap=64, bs=16, nb=4096, B=1 << 30, select=0):
    return Engine(EngineConfig(block_size=bs, num_blocks=nb, max_rows=B, T=T, cap=cap, eos_id=1,
                               select_mode=select), ScriptedSource(1))


# ------------------------------------------------------------------ hand traces
def test_trace_A_two_phase_pruning():
    scores = np.zeros((4, 4), np.float32)
    scores[:, 0] = [0.6, 0.4, 0.3, 0.45]      # boundary 16
    scores[0, 1], scores[3, 1] = 0.55, 0.2    # boundary 32
    scores[3, 2] = 0.6                        # boundary 48
    finals = [0.7, 0.0, 0.0, 0.0]
    e = engine()
    e.admit(mk_req(0, [40, 20, 64, 50], scores, finals, M=2, alpha=0.5, beta=2))
    e.step(1)                                  # boundary 16
    m = e.snapshot()["meta"][0]
    assert m[:5] == (EXPLORE, np.float32(0.5), 2, 0, 2)
    assert [r[1] for r in e.snapshot()["rows"]] == [0, 3]   # b1, b2 pruned; b3 spared by the cap
    e.step(1)                                  # boundary 32: b3 at 0.2 but cap reached
    assert [r[1] for r in e.snapshot()["rows"]] == [0, 3]
    e.step(1)                                  # boundary 48
    res = e.collect()
    assert len(res) == 1
    r = res[0]
    assert r["phase_at_end"] == EXPLOIT and r["threshold_at_end"] == np.float32(0.7)
    assert (r["num_completed"], r["num_pruned"], r["num_early_stopped"]) == (1, 3, 0)
    assert r["finalize_reason"] == 1
    assert r["branch_state"] == [COMPLETED_EOS, PRUNED, PRUNED, PRUNED]
    assert r["branch_len"] == [40, 16, 16, 48]
    assert r["chosen_max_reward"] == 0 and r["window_final"] == 2


def test_trace_B_early_stop_and_allocator():
    # SURVEY's trace uses NB=16, but commitment (R34) needs 1 + 4*4 = 17 blocks for 4 rows
    e = engine(T=16, cap=64, bs=16, nb=17)
    e.admit(mk_req(0, [30, 10, 50, 25], np.zeros((4, 4)), M=2, alpha=-1.0, beta=0, P=17))
    e._fill()
    assert e.live[0].prefix_blocks == [0]
    assert [r.blocks for r in e.rows] == [[1], [2], [3], [4]]
    assert e.free == list(range(16, 4, -1))
    e._decode_window(); e._boundary(); e.window += 1            # boundary 16
    s = e.snapshot()
    assert [r[1] for r in s["rows"]] == [0, 2, 3]
    assert s["tables"] == [[1, 2], [3, 5], [4, 6]]
    assert s["free"] == list(range(16, 6, -1))
    e.step(1)                                                    # boundary 32
    s = e.snapshot()
    assert s["free"] == list(range(16, 6, -1)) + [1, 2, 3, 5, 4, 6, 0]
    assert s["committed"] == 0 and s["rows"] == []
    r = e.collect()[0]
    assert r["branch_state"] == [COMPLETED_EOS, COMPLETED_EOS, EARLY_STOPPED, COMPLETED_EOS]
    assert r["branch_len"] == [30, 10, 32, 25]
    assert r["num_completed"] == 3 and r["finalize_reason"] == 0


# ------------------------------------------------------------------ SPEC examples
def test_spec_S271_explore_prune_hits_beta():
    rewards = [0.3, 0.6, 0.2, 0.7, 0.45, 0.9, 0.1, 0.55]
    sc = np.tile(np.asarray(rewards, np.float32)[:, None], (1, 4))
    e = engine()
    e.admit(mk_req(0, [64] * 8, sc, M=4, alpha=0.5, beta=4))
    e.step(1)
    st = e.live[0].branch_state
    assert [b for b in range(8) if st[b] == PRUNED] == [0, 2, 4, 6]   # 1-based {1,3,5,7}
    assert e.live[0].num_pruned == 4


def test_spec_S272_first_completion_sets_threshold():
    sc = np.full((4, 4), 0.9, np.float32)
    e = engine()
    e.admit(mk_req(0, [10, 64, 64, 64], sc, finals=[0.82, 0, 0, 0], M=3, alpha=0.5, beta=2))
    e.step(1)
    m = e.live[0]
    assert (m.phase, m.threshold, m.max_num_pruned, m.num_completed) == (EXPLOIT, np.float32(0.82), 3, 1)


def test_spec_S273_M_completions_early_stop():
    e = engine()
    e.admit(mk_req(0, [5, 9, 64, 64], np.full((4, 4), 0.9), finals=[0.9, 0.9, 0, 0], M=2))
    e.step(1)
    r = e.collect()[0]
    assert r["branch_state"] == [COMPLETED_EOS, COMPLETED_EOS, EARLY_STOPPED, EARLY_STOPPED]
    assert r["num_early_stopped"] == 2 and r["finalize_reason"] == 0


@pytest.mark.parametrize("labels,vote", [([0, 0, 3, 0], 0), ([1, 1, 0, 0], 1)])
def test_spec_S280_S281_vote(labels, vote):
    e = engine()
    e.admit(mk_req(0, [4, 4, 4, 4], np.zeros((4, 4)), answers=labels, M=4, alpha=-1, beta=0))
    e.step(5)
    assert e.collect()[0]["answer_vote"] == vote


def test_spec_S282_max_reward():
    e = engine(select=1)
    e.admit(mk_req(0, [4, 4, 4], np.zeros((3, 4)), finals=[0.7, 0.9, 0.8], answers=[5, 6, 7],
                   M=3, alpha=-1, beta=0))
    e.step(5)
    r = e.collect()[0]
    assert r["chosen_max_reward"] == 1 and r["answer_max_reward"] == 6 and r["selected_branch"] == 1


# ------------------------------------------------------------------ brute force vs naive Alg. 1
def naive_alg1(N, M, alpha, beta, lengths, scores, finals, T):
    """Independent transcription of Alg. 1 L21-40 for N branches that all start together
    (no allocator, no batch limit).  Returns per-branch states and the meta record."""
    phase, thr, maxp, nc, npr = "explore", np.float32(alpha), beta, 0, 0
    st = ["run"] * N
    ln = [0] * N
    t, k = 0, 0
    while True:
        live = [b for b in range(N) if st[b] == "run"]
        wend = min(t + T, max(lengths[b] for b in live))      # up to T steps; ends when none live
        done = [b for b in live if lengths[b] <= wend]
        if phase == "explore" and done:                         # L24-27
            first = min(done, key=lambda b: (lengths[b], b))
            phase, thr, maxp = "exploit", np.float32(finals[first]), N - 1
        for b in done:                                          # L28-31
            st[b], ln[b] = "C", lengths[b]
            nc += 1
        if alpha >= 0:
            for b in sorted(set(live) - set(done)):             # L32-37
                if npr < maxp and np.float32(scores[b][k]) < thr:
                    st[b], ln[b] = "P", wend
                    npr += 1
        if nc >= M or nc + npr == N:                            # L38-40
            for b in range(N):
                if st[b] == "run":
                    st[b], ln[b] = "ES", wend
            return st, ln, phase, thr, nc, npr
        t, k = wend, k + 1


def test_brute_force_vs_naive_and_predicates():
    rng = np.random.default_rng(7)
    T = 4
    code = {COMPLETED_EOS: "C", PRUNED: "P", EARLY_STOPPED: "ES"}
    n_cases = 0
    for N in range(1, 5):
        for M in range(1, N + 1):
            for beta in range(0, N):
                for _ in range(60 if N == 4 else 40):
                    lengths = [int(x) * T for x in rng.integers(1, 4, N)]
                    scores = rng.choice([0.25, 0.75], size=(N, 3)).astype(np.float32)
                    finals = rng.choice([0.25, 0.75], size=N).astype(np.float32)
                    alpha = 0.5 if rng.random() < 0.85 else -1.0
                    e = engine(T=T, cap=3 * T)
                    e.admit(mk_req(0, lengths, scores, finals, M=M, alpha=alpha, beta=beta))
                    e.step(100)
                    r = e.collect()[0]
                    st, ln, phase, thr, nc, npr = naive_alg1(N, M, alpha, beta, lengths, scores,
                                                             finals, T)
                    assert [code[s] for s in r["branch_state"]] == st
                    assert r["branch_len"] == ln
                    assert (r["num_completed"], r["num_pruned"]) == (nc, npr)
                    assert r["threshold_at_end"] == thr
                    # predicates the paper fixes
                    assert r["num_pruned"] <= (beta if r["phase_at_end"] == EXPLORE else N - 1)
                    assert r["num_completed"] >= M or r["num_completed"] + r["num_pruned"] == N
                    assert (r["num_completed"] + r["num_pruned"] + r["num_early_stopped"]
                            + r["num_discarded_queued"]) == N
                    assert r["num_completed"] >= 1
                    if alpha < 0:
                        assert r["num_pruned"] == 0
                    n_cases += 1
    assert n_cases > 1000


# ------------------------------------------------------------------ allocator invariants
def check_invariants(e):
    cfg = e.cfg
    owned = []
    for r in e.rows:
        assert len(r.blocks) == -(-min(r.ell + cfg.T, cfg.cap) // cfg.block_size)
        owned += r.blocks
    for rs in e.live.values():
        owned += rs.prefix_blocks
    allb = owned + e.free
    assert len(allb) == len(set(allb)) == cfg.num_blocks           # disjoint and complete
    rc = -(-cfg.cap // cfg.block_size)
    commit = len(e.rows) * rc + sum(-(-(rs.P - 1) // cfg.block_size) for rs in e.live.values())
    assert commit == e.committed <= cfg.num_blocks                  # ledger recompute
    assert len(e.rows) <= cfg.max_rows


@pytest.mark.parametrize("seed", range(12))
def test_allocator_invariants_random(seed):
    rng = np.random.default_rng(seed)
    bs = int(rng.choice([16, 64]))
    T = int(rng.choice([1, 4, 16]))
    cap = int(rng.integers(8, 200))
    N = int(rng.integers(1, 9))
    M = int(rng.integers(1, N + 1))
    shape = SHAPES["tiny"]
    reqs = gen_requests(int(rng.integers(3, 9)), shape, N, M, 0.5 if rng.random() < 0.7 else -1.0,
                        int(rng.integers(0, N)), cap, T, eos_id=1, p_range=(1, 150),
                        length="uniform", len_range=(1, cap), root_seed=seed)
    need = max(-(-(len(r.prompt) - 1) // bs) for r in reqs) + -(-cap // bs)
    nb = int(need + rng.integers(0, 3 * need))
    B = int(rng.integers(1, 3 * N + 1)) if rng.random() < 0.5 else 1 << 30
    e = engine(T=T, cap=cap, bs=bs, nb=nb, B=B)
    for r in reqs:
        e.admit(r)
    for _ in range(10_000):
        before = e.window
        e.step(1)
        check_invariants(e)
        if e.window == before:
            break
    res = e.collect()
    assert sorted(r["request_id"] for r in res) == [r.request_id for r in reqs]
    assert len(e.free) == nb and e.committed == 0                    # drained: all blocks free
    assert sorted(e.free) == list(range(nb))
    # FCFS: finalization of prefills follows arrival order of prefill
    for r in res:
        assert r["num_completed"] >= 1


# ------------------------------------------------------------------ vote
def plurality(labels):
    counts = collections.Counter(labels)
    best = max(counts.values())
    cands = [lab for lab in counts if counts[lab] == best]
    return min(cands, key=lambda lab: labels.index(lab)), best


def test_vote_exhaustive():
    for N in range(1, 6):
        for labels in itertools.product(range(3), repeat=N):
            e = engine()
            e.admit(mk_req(0, [3] * N, np.zeros((N, 4)), answers=list(labels), M=N, alpha=-1,
                           beta=0))
            e.step(3)
            r = e.collect()[0]
            assert (r["answer_vote"], r["vote_count"]) == plurality(list(labels))


# ------------------------------------------------------------------ degenerate policies
def test_vanilla_equivalence():
    """SART with N = M = 1, alpha = 0, beta = 0 is Vanilla: the single branch runs
    to its own length, nothing is pruned."""
    for L in [1, 5, 16, 17, 63, 64]:
        e = engine()
        e.admit(mk_req(0, [L], np.zeros((1, 4)), finals=[0.0], M=1, alpha=0.0, beta=0))
        e.step(100)
        r = e.collect()[0]
        assert e.steps == L and r["branch_state"] == [COMPLETED_EOS if L < 64 or True else 0]
        assert r["branch_len"] == [L] and r["num_pruned"] == 0


def test_self_consistency_equivalence():
    """M = N with pruning disabled waits for all N completions."""
    e = engine()
    e.admit(mk_req(0, [10, 64, 33, 5], np.zeros((4, 4)), M=4, alpha=-1.0, beta=0))
    e.step(100)
    r = e.collect()[0]
    assert r["num_completed"] == 4 and e.steps == 64
    assert r["branch_state"][1] == COMPLETED_EOS        # forced EOS at the cap step is EOS


def test_cap_counts_as_completion():
    """R17: a branch reaching the cap without EOS is Completed (reason CAP)."""
    e = engine(cap=20)
    e.admit(mk_req(0, [30, 8], np.zeros((2, 4)), M=2, alpha=-1.0, beta=0))
    e.step(100)
    r = e.collect()[0]
    assert r["branch_state"] == [COMPLETED_CAP, COMPLETED_EOS] and r["branch_len"] == [20, 8]


def test_queued_branches_discarded_and_fcfs():
    """B smaller than N: queued branches of a finalized request are Discarded (R7)."""
    e = engine(B=2)
    e.admit(mk_req(0, [3, 3, 64, 64], np.zeros((4, 4)), M=2, alpha=-1.0, beta=0))
    e.admit(mk_req(1, [5, 5], np.zeros((2, 4)), M=1, alpha=-1.0, beta=0))
    e.step(100)
    res = e.collect()
    assert [r["request_id"] for r in res] == [0, 1]
    assert res[0]["branch_state"] == [COMPLETED_EOS, COMPLETED_EOS, DISCARDED, DISCARDED]
    assert res[0]["num_discarded_queued"] == 2


def test_prm_model_source_scores_the_read_prefix():
    """Row f2 (reading R42): with a separate PRM model, every completed branch's final score
    is the PRM's score of prompt + y_1 .. y_{len-1}, computed by one uncached forward; the
    pool drains back to full."""
    from oracle.engine import ModelSource
    from oracle.model import Model
    from synth import gen_prompt, gen_weights
    pol, prm = SHAPES["tiny"], SHAPES["prm-tiny"]
    cfg = EngineConfig(block_size=16, num_blocks=64, max_rows=64, T=4, cap=12, eos_id=1, temperature=1.0,
                       sampler_seed=3)
    pm = Model(prm, gen_weights(prm, "fp32", std=0.05, root_seed=91))
    prompt = gen_prompt(0, pol.vocab, 1, 5, 5)
    forced = np.random.default_rng(1).integers(2, pol.vocab, size=(3, 12)).astype(np.int32)
    forced[0, 6] = 1                                   # branch 0 emits EOS at step 7
    src = ModelSource(Model(pol, gen_weights(pol, "fp32", std=0.05)), cfg, prm_model=pm,
                      forced_tokens={0: forced})
    e = Engine(cfg, src)
    e.admit(Request(0, prompt, 3, 3, -1.0, 0, None))
    e.step(100)
    r = e.collect()[0]
    assert r["branch_len"] == [7, 12, 12] and r["num_completed"] == 3
    for b in range(3):
        L = r["branch_len"][b]
        seq = [int(t) for t in prompt] + [int(t) for t in forced[b, : L - 1]]
        assert r["branch_score"][b] == np.float32(pm.prm_model_score(seq))
    assert e.stats()["free_blocks"] == 64


# ------------------------------------------------------------------ R44: interleaved prefill
def _engine_pc(T, cap, pc, bs=16, nb=4096, B=1 << 30):
    return Engine(EngineConfig(block_size=bs, num_blocks=nb, max_rows=B, T=T, cap=cap, eos_id=1,
                               prefill_chunk=pc), ScriptedSource(1))


def test_interleaved_prefill_start_steps():
    """Three requests prefilled in one fill with 10, 25 and 5 prefix tokens and 16-token chunks:
    the batch is [0, 10) [10, 35) [35, 40), chunks [0,16) [16,32) [32,48) run before steps 1,
    2, 3, so the requests' rows start at steps 1, 3 and 3 and have 8, 6, 6 tokens after an
    8-step window (lengths longer than the window, pruning off)."""
    e = _engine_pc(T=8, cap=64, pc=16)
    for rid, P in enumerate((11, 26, 6)):
        e.admit(mk_req(rid, [50, 50], np.zeros((2, 8)), M=2, alpha=-1.0, beta=0, P=P))
    e.step(1)
    ells = {(r[0], r[1]): r[2] for r in e.snapshot()["rows"]}
    assert ells == {(0, 0): 8, (0, 1): 8, (1, 0): 6, (1, 1): 6, (2, 0): 6, (2, 1): 6}
    e.step(1)                                   # the next window starts every row at step 1
    assert {(r[0], r[1]): r[2] for r in e.snapshot()["rows"]} == {k: v + 8 for k, v in ells.items()}


def test_interleaved_prefill_one_chunk_equals_inline():
    """A chunk that holds every fill's whole batch is inline prefill: identical snapshots and
    records on random scripted workloads."""
    rng = np.random.default_rng(44)
    for seed in range(4):
        reqs = gen_requests(8, SHAPES["tiny"], 4, 2, 0.5, 2, 48, 8, eos_id=1, p_range=(2, 60), length="uniform",
                            len_range=(1, 48), root_seed=seed)
        a, b = _engine_pc(8, 48, 0, nb=120, B=12), _engine_pc(8, 48, 10 ** 6, nb=120, B=12)
        for r in reqs:
            a.admit(r)
            b.admit(r)
        for _ in range(200):
            a.step(1)
            b.step(1)
            assert a.snapshot() == b.snapshot()
        assert a.collect() == b.collect()


def test_interleaved_prefill_keeps_branch_lengths():
    """With M = N and pruning off every branch completes at its scripted length, whatever step
    it starts at: interleaving changes when rows decode, never what they decode."""
    for pc in (4, 16, 64):
        e = _engine_pc(T=6, cap=40, pc=pc, nb=400, B=10)
        reqs = gen_requests(6, SHAPES["tiny"], 3, 3, -1.0, 0, 40, 6, eos_id=1, p_range=(10, 90), length="uniform",
                            len_range=(1, 40), root_seed=pc)
        for r in reqs:
            e.admit(r)
        e.step(1000)
        res = {x["request_id"]: x for x in e.collect()}
        for r in reqs:
            assert res[r.request_id]["branch_len"] == [int(x) for x in r.script.forced_len]
