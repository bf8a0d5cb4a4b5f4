"""Request-partitioned multi-GPU serving.

Requests are independent (all bookkeeping is per request), so the hot path
shards by request: one process and one engine per GPU, full weight replica per GPU, no KV
or activation traffic between GPUs.  The only collectives are

  C1  an all-gather of a fixed int32[16] counter record per rank at every window boundary
      (used by the least-loaded dispatcher; 64 B per rank), and
  C2  a gather of the finished result records to rank 0.

Both go through torch.distributed (NCCL on GPUs, gloo in the CPU tests).  Dispatch is
computed identically on every rank from the gathered counters, so no extra messages are
needed and per-rank replays stay deterministic.

The engine is duck-typed: ``admit(req)``, ``step(n) -> stats dict``, ``collect() -> list``
and ``counters(out) -> torch.int32[16]``: the CUDA engine (``sart.Engine``) fills the device
tensor ``out`` with ``sart_export_counters``; a host stand-in may ignore ``out`` and return a
CPU tensor (gloo).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence

import torch
import torch.distributed as dist

# fields of the C1 record (sart_export_counters order)
LIVE_ROWS, QUEUED_BRANCHES, QUEUED_REQUESTS, FREE_BLOCKS, COMMITTED, FINALIZED, WINDOWS, STEPS = range(8)


def round_robin(requests: Sequence, rank: int, world: int) -> List:
    """Static partition by arrival index (deterministic; per-rank oracle replay stays exact)."""
    return list(requests[rank::world])


class LeastLoaded:
    """Least-loaded dispatch from the all-gathered counters: fewest queued requests (plus the
    ones assigned since the last gather), then fewest committed blocks, then lowest rank."""

    def __init__(self, world: int):
        self.world = world
        self.pending = [0] * world

    def assign(self, counters: torch.Tensor, n_new: int) -> List[int]:
        c = counters.to("cpu").tolist()
        load = [(c[r][QUEUED_REQUESTS] + self.pending[r], c[r][COMMITTED], r) for r in range(self.world)]
        out = []
        for _ in range(n_new):
            best = min(range(self.world), key=lambda r: load[r])
            out.append(best)
            q, cm, r = load[best]
            load[best] = (q + 1, cm, r)
            self.pending[best] += 1
        return out

    def gathered(self):
        self.pending = [0] * self.world


def all_gather_counters(mine: torch.Tensor, group=None) -> torch.Tensor:
    """C1: every rank's int32[16] record -> [world, 16] on every rank."""
    world = dist.get_world_size(group)
    out = torch.empty(world * mine.numel(), dtype=mine.dtype, device=mine.device)
    dist.all_gather_into_tensor(out, mine.contiguous().view(-1), group=group)
    return out.view(world, -1)


def gather_results(results: List[Dict], group=None, dst: int = 0) -> List[Dict]:
    """C2: result records of all ranks -> rank dst (ordered by request_id there)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bucket = [None] * world if rank == dst else None
    dist.gather_object(results, bucket, dst=dst, group=group)
    if rank != dst:
        return []
    merged = [r for part in bucket for r in part]
    return sorted(merged, key=lambda r: r["request_id"])


# C2 with fixed-size records: one int32 row per finalized request, gathered to rank 0 by the
# backend's own collectives (NCCL over NVLink on GPUs) instead of pickled objects.
RECORD_FIELDS = ("request_id", "answer_vote", "vote_count", "chosen_max_reward", "answer_max_reward",
                 "num_completed", "num_pruned", "num_early_stopped", "num_discarded_queued", "finalize_reason",
                 "phase_at_end", "window_final", "selected_branch", "tokens_len")


def gather_result_records(results: List[Dict], device, group=None, dst: int = 0) -> torch.Tensor:
    """C2: every rank's result records as int32 rows [len(RECORD_FIELDS)] (request_id must
    fit int32) -> rank dst gets [total, F] ordered by rank then finalization order; other ranks
    get an empty tensor.  Two all-gathers: the per-rank counts, then the rows padded to the
    largest count."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    F = len(RECORD_FIELDS)
    rows = [[int(r[k]) if k != "tokens_len" else int(r.get(k, len(r.get("tokens", ())))) for k in RECORD_FIELDS]
            for r in results]
    mine = (torch.tensor(rows, dtype=torch.int32) if rows else torch.zeros((0, F), dtype=torch.int32)).to(device)
    cnt = torch.tensor([mine.shape[0]], dtype=torch.int32, device=device)
    cnts = torch.zeros(world, dtype=torch.int32, device=device)
    dist.all_gather_into_tensor(cnts, cnt, group=group)
    mx = int(cnts.max().item())
    pad = torch.zeros((max(mx, 1), F), dtype=torch.int32, device=device)
    pad[: mine.shape[0]] = mine
    allr = torch.zeros((world * max(mx, 1), F), dtype=torch.int32, device=device)
    dist.all_gather_into_tensor(allr, pad, group=group)
    if rank != dst:
        return torch.zeros((0, F), dtype=torch.int32)
    allr = allr.view(world, max(mx, 1), F).cpu()
    return torch.cat([allr[r, : int(cnts[r])] for r in range(world)], 0)


def serve(engine, arrivals: Sequence[Sequence], policy: str = "round_robin", group=None,
          max_windows: int = 1 << 30, on_window: Callable = None) -> List[Dict]:
    """Run a request stream to completion on this rank.

    arrivals[w] is the list of requests that arrive before window w (the same global list on
    every rank).  Round-robin assigns the k-th arrival overall to rank k % world; least-loaded
    assigns each window's arrivals from the counters gathered at the previous boundary.
    Returns this rank's finished results (use gather_results for rank 0's view).
    """
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ll = LeastLoaded(world)
    backend = dist.get_backend(group)
    # the C1 record lives where the backend's collectives read it: the rank's GPU for NCCL
    cbuf = torch.zeros(16, dtype=torch.int32,
                       device=f"cuda:{torch.cuda.current_device()}" if backend == "nccl" else "cpu")
    counters = None
    k = 0
    results: List[Dict] = []
    w = 0
    while w < max_windows:
        new = arrivals[w] if w < len(arrivals) else []
        if policy == "round_robin":
            owners = [(k + i) % world for i in range(len(new))]
        else:
            if counters is None:
                counters = torch.zeros((world, 16), dtype=torch.int32)
            owners = ll.assign(counters, len(new))
        k += len(new)
        for req, o in zip(new, owners):
            if o == rank:
                engine.admit(req)
        st = engine.step(1)
        results += engine.collect()
        counters = all_gather_counters(engine.counters(cbuf), group)
        ll.gathered()
        if on_window:
            on_window(w, st, counters)
        w += 1
        idle = counters[:, LIVE_ROWS].sum() + counters[:, QUEUED_BRANCHES].sum() + counters[:, QUEUED_REQUESTS].sum()
        if w >= len(arrivals) and int(idle) == 0:
            break
    return results
