"""Algorithm 1 of PAPER as a step-by-step CPU engine.

Written in the paper's order and notation; every choice the paper leaves open
is a numbered reading in DESIGN.md ("R<n>").  Line references "L<k>" are
Algorithm 1's own line numbers (map in SURVEY §8(c)).

Main loop (L1-13):
    while not terminated:
        while len(current_batch) < B:                               L3
            if branch_queue: current_batch.append(branch_queue.pop())  L4-5
            elif request_queue: Prefill(request_queue.pop())           L6-7
            else: break                                                L8-9
        Decode(current_batch, T)                                       L12

Prefill(i) (L14-20): meta[i] = {explore, alpha, beta, 0, 0}; push b_i1..b_iN.
Decode (L21-40): up to T batched steps, then per involved request:
    L24-27 phase switch on the first completion (alpha' = its reward, cap N-1)
    L28-31 completed branches removed, num_completed += 1
    L32-37 prune incomplete branches with PRM < threshold while num_pruned < max
    L38-40 output when num_completed >= M or num_completed + num_pruned == N

Readings used here: R2 first completion = smallest window step,
ties -> lowest branch; R3 alpha' literal; R4 prune in ascending branch index;
R5 strict '<'; R6 switch before prune; R7 finalize early-stops running rows
and discards queued branches; R8 control only at T boundaries; R9 slots and
blocks released at the boundary; R17 cap counts as completion; R18 FIFO
queues; R19 involved = >= 1 row in this window's batch; R20 alpha < 0
disables pruning in both phases; R21 ascending request_id; R23 block
allocator (LIFO free stack, O8 order); R31 a window ends early when no row
is live; R34 commitment admission.

Block allocator and commitment (R23, R34 -- our proposal, the paper
delegates paging to vLLM; prefix shared and freed only when all
branches ended):
    initial free stack bottom->top [NB-1, ..., 1, 0]
    boundary: (1) free terminated rows' suffix blocks in batch-row order and
              logical order, then prefix blocks of requests finalized at this
              boundary in ascending request_id; (2) stable compaction;
              (3) reserve: each surviving row owns ceil(min(l+T, cap)/bs) blocks
    admission: a prefill pops ceil((P-1)/bs) prefix blocks; a new row pops
              ceil(min(T, cap)/bs) blocks
    committed = sum_live_requests ceil((P-1)/bs) + sum_live_rows ceil(cap/bs)
    admission requires committed + new <= NB (prefill: prefix + one row).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import collections
import dataclasses
from typing import Dict, List, Optional

import numpy as np

from . import philox
from .model import Model

# branch states (also the values of sart_result.branch_state)
QUEUED, RUNNING, COMPLETED_EOS, COMPLETED_CAP, PRUNED, EARLY_STOPPED, DISCARDED = range(7)
EXPLORE, EXPLOIT = 0, 1


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def f32(x) -> float:
    return float(np.float32(x))


@dataclasses.dataclass
class EngineConfig:
    block_size: int = 64
    num_blocks: int = 1024
    max_rows: int = 1 << 30       # B
    T: int = 400                  # ctl_interval (default)
    cap: int = 4096               # max_new_tokens
    eos_id: int = 1
    temperature: float = 1.0
    sampler_seed: int = 0
    select_mode: int = 0          # 0 = vote, 1 = max reward (which branch's tokens are returned)
    # Reading R43 (variant of R8): once a request has M completed branches,
    # its other running branches stop decoding at that step; they are EarlyStopped at the
    # boundary (never pruned).  False = paper semantics: early stop only at T boundaries.
    es_every_step: bool = False
    # Reading R44 (row f1): 0 = each fill's prefill runs before the window's first decode step
    # (Alg. 1 L7 inline).  C > 0 = chunked prefill interleaved with decode: the fill's prompts
    # (prefix tokens, FCFS order, concatenated) are processed in C-token chunks, chunk c right
    # before window step min(c + 1, T); the rows of a request prefilled in this fill start
    # decoding at the step whose chunk completes its prefix, the other rows at step 1.
    prefill_chunk: int = 0


@dataclasses.dataclass
class ReqState:
    req: object                   # synth.Request
    rid: int
    N: int
    M: int
    P: int
    alpha: float
    beta: int
    prune_enabled: bool
    phase: int = EXPLORE
    threshold: float = 0.0
    max_num_pruned: int = 0
    num_completed: int = 0
    num_pruned: int = 0
    num_early_stopped: int = 0
    num_discarded: int = 0
    prefix_blocks: List[int] = dataclasses.field(default_factory=list)
    branch_state: List[int] = dataclasses.field(default_factory=list)
    branch_len: List[int] = dataclasses.field(default_factory=list)
    branch_score: List[float] = dataclasses.field(default_factory=list)
    branch_label: List[int] = dataclasses.field(default_factory=list)
    branch_tokens: Dict[int, List[int]] = dataclasses.field(default_factory=dict)
    window_prefill: int = -1
    ready_wstep: int = 1          # R44: window step at which its prefix is complete (window_prefill)


@dataclasses.dataclass
class Row:
    rs: ReqState
    b: int                        # the paper's j in b_ij (0-based)
    ell: int = 0                  # decode steps done = tokens generated (R22)
    running: bool = True
    reason: int = 0               # COMPLETED_EOS / COMPLETED_CAP when done
    done_step: int = 0
    done_wstep: int = 0
    nbnd: int = 0                 # boundaries seen while running (script index k)
    score: float = 0.0
    blocks: List[int] = dataclasses.field(default_factory=list)
    hist: List[int] = dataclasses.field(default_factory=list)
    terminal: int = RUNNING       # state decided at the boundary
    stopped: bool = False         # R43: stopped mid-window by early stop (incomplete)
    start: int = 1                # R44: first window step this row decodes in its first window


# ------------------------------------------------------------------ sources
class ScriptedSource:
    """Tokens and rewards from a synth.Script.

    EOS is emitted exactly at step forced_len; the other token values do not
    influence control, so they are not produced (placeholder -1).  Score at
    the k-th boundary a branch is running at: scores[b][min(k, n_bnd-1)]
    (reading R35); final score at completion: final_score[b]."""

    def __init__(self, eos_id: int):
        self.eos = eos_id

    def on_prefill(self, rs: ReqState):
        pass

    def step(self, rows: List[Row], wstep: int) -> List[int]:
        out = []
        for r in rows:
            s = r.ell + 1
            out.append(self.eos if s == int(r.rs.req.script.forced_len[r.b]) else -1)
        return out

    def score_running(self, r: Row, k: int) -> float:
        sc = r.rs.req.script.scores
        return f32(sc[r.b, min(k, sc.shape[1] - 1)])

    def score_final(self, r: Row) -> float:
        return f32(r.rs.req.script.final_score[r.b])


class ModelSource:
    """Free-running model mode: oracle Model + Philox/Gumbel sampler + PRM head.
    A request with a script keeps its forced EOS step (O4) and script scores
    unless ``prm_scores`` is set."""

    def __init__(self, model: Model, cfg: EngineConfig, prm_scores: bool = True,
                 prm_model: Optional[Model] = None, forced_tokens: Optional[dict] = None):
        self.m = model
        self.cfg = cfg
        self.prm = prm_scores
        self.prm_model = prm_model      # row f2: separate PRM decoder (else the head on z)
        self.forced = forced_tokens or {}   # teacher forcing: {rid: int[N][cap]}, y_s := [b][s-1]
        self.prefix = {}
        self.suffix = {}
        self.z = {}

    def on_prefill(self, rs: ReqState):
        self.prefix[rs.rid] = self.m.prefill(rs.req.prompt)

    def step(self, rows: List[Row], wstep: int) -> List[int]:
        toks, pos, pre, suf = [], [], [], []
        for r in rows:
            s = r.ell + 1
            key = (r.rs.rid, r.b)
            if key not in self.suffix:
                self.suffix[key] = [{"k": [], "v": []} for _ in range(self.m.s.n_layers)]
            toks.append(int(r.rs.req.prompt[-1]) if s == 1 else r.hist[-1])
            pos.append(r.rs.P - 2 + s)
            pre.append(self.prefix[r.rs.rid])
            suf.append(self.suffix[key])
        z, logits = self.m.decode(np.array(toks), np.array(pos), pre, suf)
        out = []
        for i, r in enumerate(rows):
            self.z[(r.rs.rid, r.b)] = z[i]
            sc = r.rs.req.script
            forced = int(sc.forced_len[r.b]) if sc is not None else 0
            y = philox.sample(logits[i].astype(np.float32), r.ell + 1, r.rs.rid, r.b,
                              self.cfg.sampler_seed, self.cfg.temperature, self.cfg.eos_id, forced)
            if r.rs.rid in self.forced:       # teacher forcing replaces the sampled token
                y = int(self.forced[r.rs.rid][r.b][r.ell])
            out.append(y)
        return out

    def _prm(self, r: Row) -> float:
        if self.prm_model is not None:
            # row f2, reading R42: the PRM reads prompt + y_1 .. y_{l-1} (the tokens whose
            # policy KV entries exist) and scores the last of them
            seq = list(int(t) for t in r.rs.req.prompt) + list(r.hist[: r.ell - 1])
            return f32(self.prm_model.prm_model_score(seq))
        return f32(self.m.prm_score(self.z[(r.rs.rid, r.b)])[0])

    def score_running(self, r: Row, k: int) -> float:
        if self.prm or r.rs.req.script is None:
            return self._prm(r)
        return ScriptedSource.score_running(self, r, k)

    def score_final(self, r: Row) -> float:
        if self.prm or r.rs.req.script is None:
            return self._prm(r)
        return ScriptedSource.score_final(self, r)


class ReplaySource:
    """Replays recorded token and score streams (PP2): tokens[(rid, b)][s-1],
    running[(rid, b)][k] and final[(rid, b)] (fp32 values)."""

    def __init__(self, tokens: dict, running: dict, final: dict):
        self.tokens, self.running, self.final = tokens, running, final

    def on_prefill(self, rs):
        pass

    def step(self, rows, wstep):
        return [int(self.tokens[(r.rs.rid, r.b)][r.ell]) for r in rows]

    def score_running(self, r, k):
        return f32(self.running[(r.rs.rid, r.b)][k])

    def score_final(self, r):
        return f32(self.final[(r.rs.rid, r.b)])


# ------------------------------------------------------------------ engine
class Engine:
    def __init__(self, cfg: EngineConfig, source):
        self.cfg = cfg
        self.src = source
        self.free: List[int] = list(range(cfg.num_blocks - 1, -1, -1))  # bottom -> top
        self.committed = 0
        self.rows: List[Row] = []
        self.request_queue: collections.deque = collections.deque()
        self.branch_queue: collections.deque = collections.deque()
        self.live: Dict[int, ReqState] = {}
        self.results: List[dict] = []
        self.window = 0
        self.steps = 0
        self.branch_tokens = 0
        self.finalized_total = 0
        self.seen_ids = set()

    # -------------------------------------------------------------- helpers
    def _pop(self, n: int) -> List[int]:
        out = []
        for _ in range(n):
            assert self.free, "free stack underflow (commitment violated)"
            out.append(self.free.pop())
        return out

    def row_commit(self) -> int:
        return cdiv(self.cfg.cap, self.cfg.block_size)

    def prefix_commit(self, P: int) -> int:
        return cdiv(P - 1, self.cfg.block_size)

    # -------------------------------------------------------------- intake
    def admit(self, req) -> None:
        """request_queue.push; validation mirrors include/sart.h."""
        N, M = req.N, req.M
        if not (1 <= M <= N <= 32):
            raise ValueError("EINVAL: need 1 <= M <= N <= 32")
        beta = N // 2 if req.beta == -1 else req.beta
        if not (0 <= beta <= N - 1):
            raise ValueError("EINVAL: beta")
        if not (req.alpha <= 1.0) or np.isnan(req.alpha):
            raise ValueError("EINVAL: alpha")
        if len(req.prompt) < 1:
            raise ValueError("EINVAL: prompt")
        if req.request_id in self.seen_ids:
            raise ValueError("EDUP")
        if self.prefix_commit(len(req.prompt)) + self.row_commit() > self.cfg.num_blocks:
            raise MemoryError("ENOMEM: request can never be admitted")
        self.seen_ids.add(req.request_id)
        self.request_queue.append(req)

    # -------------------------------------------------------------- Prefill (L14-20)
    def _prefill(self, req) -> None:
        P = len(req.prompt)
        beta = req.N // 2 if req.beta == -1 else req.beta
        rs = ReqState(req=req, rid=req.request_id, N=req.N, M=req.M, P=P, alpha=f32(req.alpha),
                      beta=beta, prune_enabled=req.alpha >= 0)
        # L16: meta[i] <- {phase=explore, threshold=alpha, max_num_pruned=beta, 0, 0}
        rs.phase, rs.threshold, rs.max_num_pruned = EXPLORE, f32(req.alpha), beta
        rs.branch_state = [QUEUED] * req.N
        rs.branch_len = [0] * req.N
        rs.branch_score = [0.0] * req.N
        rs.branch_label = [-1] * req.N
        npre = self.prefix_commit(P)
        self.committed += npre
        rs.prefix_blocks = self._pop(npre)
        rs.window_prefill = self.window
        self.live[rs.rid] = rs
        self.src.on_prefill(rs)                       # L15 perform prefilling
        for j in range(req.N):                        # L17-19 push b_i1..b_iN
            self.branch_queue.append((rs, j))

    # -------------------------------------------------------------- fill loop (L3-11)
    def _fill(self) -> None:
        cfg = self.cfg
        pf_tok = 0                      # prefix tokens prefilled so far in this fill (R44)
        while len(self.rows) < cfg.max_rows:                                       # L3
            if self.branch_queue:                                                  # L4
                rs, j = self.branch_queue[0]
                if self.committed + self.row_commit() > cfg.num_blocks:
                    break                                                          # R34: no skipping
                self.branch_queue.popleft()                                        # L5
                self.committed += self.row_commit()
                row = Row(rs=rs, b=j)
                if rs.window_prefill == self.window:          # R44: after its prefix is complete
                    row.start = rs.ready_wstep
                row.blocks = self._pop(cdiv(min(cfg.T, cfg.cap), cfg.block_size))
                rs.branch_state[j] = RUNNING
                self.rows.append(row)
            elif self.request_queue:                                               # L6
                req = self.request_queue[0]
                need = self.prefix_commit(len(req.prompt)) + self.row_commit()
                if self.committed + need > cfg.num_blocks:
                    break
                self.request_queue.popleft()
                self._prefill(req)                                                 # L7
                P = len(req.prompt)
                pf_tok += P - 1
                if cfg.prefill_chunk > 0 and P > 1:   # R44: the chunk holding its last prefix token
                    self.live[req.request_id].ready_wstep = min((pf_tok - 1) // cfg.prefill_chunk + 1, cfg.T)
            else:
                break                                                              # L8-9

    # -------------------------------------------------------------- Decode (L21-40)
    def _decode_window(self) -> int:
        cfg = self.cfg
        wstep = 0
        for wstep in range(1, cfg.T + 1):                                          # L22
            if cfg.es_every_step and wstep > 1:
                self._es_stop(wstep)
                if not any(r.running for r in self.rows):                         # R31
                    break
            run = [r for r in self.rows if r.running and r.start <= wstep]
            ys = self.src.step(run, wstep)
            for r, y in zip(run, ys):
                s = r.ell + 1
                r.hist.append(int(y))
                r.ell = s
                self.branch_tokens += 1
                if y == cfg.eos_id:                   # R17 / O5
                    r.running, r.reason = False, COMPLETED_EOS
                elif s == cfg.cap:
                    r.running, r.reason = False, COMPLETED_CAP
                if not r.running:
                    r.done_step, r.done_wstep = s, wstep
            self.steps += 1
            if not any(r.running for r in self.rows):                             # R31
                break
        for r in self.rows:          # R44: later windows start every row at step 1
            r.start = 1
        return wstep

    def _es_stop(self, wstep: int) -> None:
        """R43 (es_every_step): at the start of window step wstep > 1, a running row whose
        request already has M completed branches (earlier boundaries + this window so far)
        stops; it keeps its l steps and is EarlyStopped at the boundary.  At the boundary
        itself Alg. 1's order applies (prune L32-37, then finalize L38-40)."""
        done_now = collections.Counter(r.rs.rid for r in self.rows if not r.running and not r.stopped)
        for r in self.rows:
            if r.running and r.rs.num_completed + done_now[r.rs.rid] >= r.rs.M:
                r.running, r.stopped = False, True
                r.done_step, r.done_wstep = r.ell, wstep - 1

    def _label(self, rs: ReqState, r: Row) -> int:
        sc = rs.req.script
        if sc is not None and sc.answer is not None:
            return int(sc.answer[r.b])
        for t in reversed(r.hist):                    # R16: last non-EOS token
            if t != self.cfg.eos_id:
                return int(t)
        return -1

    def _boundary(self) -> None:
        cfg = self.cfg
        # PRM scores (L25/L33): final reward for rows done this window, current otherwise
        for r in self.rows:
            if r.running or r.stopped:                # incomplete: its k-th running score
                r.score = self.src.score_running(r, r.nbnd)
                r.nbnd += 1
            else:
                r.score = self.src.score_final(r)
        involved = sorted({r.rs.rid for r in self.rows})                           # L23, R19, R21
        finalized: List[ReqState] = []
        for rid in involved:
            rs = self.live[rid]
            mine = [r for r in self.rows if r.rs is rs]
            done = [r for r in mine if not r.running and not r.stopped]
            # L24-27 phase switch (R2, R3, R6)
            if rs.phase == EXPLORE and done:
                first = min(done, key=lambda r: (r.done_wstep, r.b))
                rs.threshold = first.score
                rs.max_num_pruned = rs.N - 1
                rs.phase = EXPLOIT
            # L28-31 completed branches
            for r in done:
                r.terminal = r.reason
                rs.num_completed += 1
                rs.branch_state[r.b] = r.reason
                rs.branch_len[r.b] = r.done_step
                rs.branch_score[r.b] = r.score
                rs.branch_label[r.b] = self._label(rs, r)
                rs.branch_tokens[r.b] = list(r.hist)
            # L32-37 prune incomplete branches (R4 ascending index, R5 strict, R20)
            if rs.prune_enabled:
                for r in sorted((r for r in mine if r.running), key=lambda r: r.b):
                    if rs.num_pruned < rs.max_num_pruned and r.score < rs.threshold:
                        r.terminal = PRUNED
                        rs.num_pruned += 1
                        rs.branch_state[r.b] = PRUNED
                        rs.branch_len[r.b] = r.ell
                        rs.branch_score[r.b] = r.score
            # R43: a request with stopped rows has num_completed >= M, so it finalizes now
            assert not any(r.stopped for r in mine) or rs.num_completed >= rs.M
            # L38-40 output (R7)
            if rs.num_completed >= rs.M or rs.num_completed + rs.num_pruned == rs.N:
                for r in mine:
                    if (r.running or r.stopped) and r.terminal == RUNNING:
                        r.terminal = EARLY_STOPPED
                        rs.num_early_stopped += 1
                        rs.branch_state[r.b] = EARLY_STOPPED
                        rs.branch_len[r.b] = r.ell
                        rs.branch_score[r.b] = r.score
                keep = collections.deque()
                for item in self.branch_queue:
                    if item[0] is rs:
                        rs.num_discarded += 1
                        rs.branch_state[item[1]] = DISCARDED
                    else:
                        keep.append(item)
                self.branch_queue = keep
                finalized.append(rs)
        # (1) free: terminated rows in batch-row order, then finalized prefixes by request_id
        for r in self.rows:
            if r.terminal != RUNNING:
                self.free.extend(r.blocks)
                self.committed -= self.row_commit()
        for rs in finalized:
            self.free.extend(rs.prefix_blocks)
            self.committed -= self.prefix_commit(rs.P)
        # (2) stable compaction
        self.rows = [r for r in self.rows if r.terminal == RUNNING]
        # (3) reserve the next window's blocks
        for r in self.rows:
            need = cdiv(min(r.ell + cfg.T, cfg.cap), cfg.block_size)
            r.blocks.extend(self._pop(need - len(r.blocks)))
        # results (finalization order: window, ascending request_id)
        for rs in finalized:
            self.results.append(self._record(rs))
            del self.live[rs.rid]
            self.finalized_total += 1

    def _record(self, rs: ReqState) -> dict:
        """O9: plurality vote (ties -> label of the lowest-index tied branch) and
        max final reward (ties -> lowest index) over Completed branches."""
        comp = [b for b in range(rs.N) if rs.branch_state[b] in (COMPLETED_EOS, COMPLETED_CAP)]
        assert comp, "finalized with zero completed branches (unreachable for beta <= N-1)"
        counts = collections.Counter(rs.branch_label[b] for b in comp)
        best = max(counts.values())
        vote_b = next(b for b in comp if counts[rs.branch_label[b]] == best)
        mr_b = comp[0]
        for b in comp[1:]:
            if rs.branch_score[b] > rs.branch_score[mr_b]:
                mr_b = b
        sel = vote_b if self.cfg.select_mode == 0 else mr_b
        return dict(
            request_id=rs.rid, answer_vote=rs.branch_label[vote_b], vote_count=best,
            chosen_max_reward=mr_b, answer_max_reward=rs.branch_label[mr_b],
            num_completed=rs.num_completed, num_pruned=rs.num_pruned,
            num_early_stopped=rs.num_early_stopped, num_discarded_queued=rs.num_discarded,
            finalize_reason=0 if rs.num_completed >= rs.M else 1,
            phase_at_end=rs.phase, threshold_at_end=rs.threshold,
            branch_len=list(rs.branch_len), branch_state=list(rs.branch_state),
            branch_score=list(rs.branch_score), window_final=self.window,
            selected_branch=sel, tokens=list(rs.branch_tokens[sel]))

    # -------------------------------------------------------------- public API
    def step(self, max_windows: int) -> dict:
        for _ in range(max_windows):
            self._fill()
            if not self.rows:
                break                                  # idle: nothing to decode
            self._decode_window()
            self._boundary()
            self.window += 1
        return self.stats()

    def stats(self) -> dict:
        return dict(windows=self.window, steps=self.steps, live_rows=len(self.rows),
                    queued_branches=len(self.branch_queue),
                    queued_requests=len(self.request_queue),
                    finalized_total=self.finalized_total, free_blocks=len(self.free),
                    committed_blocks=self.committed, branch_tokens=self.branch_tokens)

    def collect(self) -> List[dict]:
        out, self.results = self.results, []
        return out

    def snapshot(self) -> dict:
        """Integer/control state after the last boundary (compared bit-exactly)."""
        return dict(
            rows=[(r.rs.rid, r.b, r.ell, r.nbnd) for r in self.rows],
            tables=[list(r.blocks) for r in self.rows],
            free=list(self.free), committed=self.committed,
            meta={rid: (rs.phase, rs.threshold, rs.max_num_pruned, rs.num_completed,
                        rs.num_pruned, list(rs.prefix_blocks))
                  for rid, rs in sorted(self.live.items())},
            branch_queue=[(rs.rid, j) for rs, j in self.branch_queue],
            request_queue=[q.request_id for q in self.request_queue])
