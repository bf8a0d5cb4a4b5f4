#!/usr/bin/env python
"""Benchmark of the SART multi-branch decode hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sart|reference]

Workload (BASELINE.json configs[1], "C2"): 1.5B-shape decoder (28 layers, d=1536, GQA 12/2,
hd 128, F 8960, V 151936) in bf16 with random-init weights; requests with N=8 branches,
M=4, cap 4096 tokens, T=400, pruning off, prompts U[64,1024], scripted lognormal lengths /
labels / rewards (DESIGN.md input recipe); B = 512 rows = 64 concurrent requests, with a
FCFS backlog so that finished requests are replaced (continuous batching, Alg. 1 L3-11).
A "step" is one window: admission + T decode steps + the device boundary.  N > 1: one
process per GPU, requests partitioned round-robin, weak scaling (64 concurrent per GPU);
the only collectives are the per-window counter all-gather and the result gather (NCCL).

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "branch-tokens/s and requests/s per box at 1/2/4/8 B200; attention HBM GB/s vs peak"
C2 = dict(shape="1.5B", N=8, M=4, alpha=-1.0, beta=4, cap=4096, T=400, p_range=(64, 1024), concurrent=64,
          block_size=64)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sart", choices=["sart", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=8, help="timed oracle decode steps of the cpu_baseline leg")
    ap.add_argument("--T", type=int, default=C2["T"])
    ap.add_argument("--attn-mode", type=int, default=0)
    return ap.parse_args()


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


# ------------------------------------------------------------------ workload
def make_requests(rank: int, world: int, first: int, count: int, shape, cfg):
    from synth import gen_requests
    reqs = gen_requests(count * world, shape, cfg["N"], cfg["M"], cfg["alpha"], cfg["beta"], cfg["cap"], cfg["T"],
                        eos_id=1, p_range=cfg["p_range"], first_id=first * world)
    return reqs[rank::world]          # round-robin partition by arrival index


# ------------------------------------------------------------------ oracle (CPU) arm
def _oracle_threads():
    """BLAS threads pinned to the cores this process may use."""
    cores = len(os.sched_getaffinity(0))
    import numpy  # noqa: F401  (load the BLAS first: threadpoolctl acts on loaded libraries only)
    try:
        from threadpoolctl import threadpool_info, threadpool_limits
        lim = threadpool_limits(limits=cores)
        used = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
        return lim, cores, used
    except Exception:
        return None, cores, cores


def _timing_weights(shape):
    """Timing input only: the oracle's cost does not depend on the weight values, so the
    tensors are filled by tiling one seeded 16M-entry normal block (seconds, instead of
    drawing 1.5B normals)."""
    import numpy as np
    from synth import weight_names, weight_shapes
    blk = (np.random.default_rng(0).standard_normal(1 << 24, dtype=np.float32) * 0.02)
    w = {}
    for name, shp in weight_shapes(shape).items():
        n = int(np.prod(shp))
        a = np.resize(blk, n).reshape(shp)
        if name.endswith("norm"):
            a = a + 1.0
        w[name] = a
    return w


def oracle_c2_slice(timed: int, warmup: int):
    """BASELINE.md §4 leg 2: a C2 slice -- 1 request, N=8 branches, P=544, 1.5B shape,
    scripted lengths -- through the oracle engine (fp64 NumPy, model mode).  The first
    window holds the prefill and is not timed; then `warmup` untimed and `timed` timed decode
    steps.  Returns per-step seconds."""
    from oracle.engine import Engine as OEngine, EngineConfig, ModelSource
    from oracle.model import Model
    from synth import SHAPES, gen_requests
    shape = SHAPES[C2["shape"]]
    t0 = time.time()
    w = _timing_weights(shape)
    gen_s = time.time() - t0
    cfg = EngineConfig(block_size=64, num_blocks=4096, T=1, cap=C2["cap"], eos_id=1)
    eng = OEngine(cfg, ModelSource(Model(shape, w), cfg, prm_scores=False))
    req = gen_requests(1, shape, C2["N"], C2["M"], C2["alpha"], C2["beta"], C2["cap"], C2["T"], eos_id=1,
                       p_range=(544, 544), first_id=0)[0]
    eng.admit(req)
    t = time.perf_counter()
    eng.step(1)                                   # prefill (543 tokens) + decode step 1
    prefill_s = time.perf_counter() - t
    times = []
    for i in range(warmup + timed):
        t = time.perf_counter()
        eng.step(1)
        if i >= warmup:
            times.append(time.perf_counter() - t)
    return dict(times=times, prefill_s=prefill_s, gen_s=gen_s)


def oracle_c1_full():
    """BASELINE.md §4 leg 1: C1 in full -- tiny decoder, 1 request, N=4, M=2, cap 64, T=16,
    alpha 0.5, beta 2, model mode (sampler + PRM head) -- through the oracle engine."""
    from oracle.engine import Engine as OEngine, EngineConfig, ModelSource
    from oracle.model import Model
    from synth import SHAPES, gen_requests, gen_weights
    shape = SHAPES["tiny"]
    cfg = EngineConfig(block_size=16, num_blocks=256, T=16, cap=64, eos_id=1)
    eng = OEngine(cfg, ModelSource(Model(shape, gen_weights(shape, "bf16", std=0.02)), cfg))
    req = gen_requests(1, shape, 4, 2, 0.5, 2, 64, 16, eos_id=1, p_range=(16, 16), scripted=False)[0]
    eng.admit(req)
    t = time.perf_counter()
    st = eng.step(1000)
    el = time.perf_counter() - t
    return dict(value=st["branch_tokens"] / el, unit="branch-tokens/s", tokens=st["branch_tokens"], s=el)


def oracle_control_replay():
    """BASELINE.md §4 leg 3: control only -- the oracle's Algorithm 1 engine replaying scripted
    token/score streams (no model) on a C3-shaped slice: 8 requests, N=16, M=4, alpha 0.5,
    beta 8, cap 8192, T=400 (the GPU's per-rank share of C3 is 32 requests)."""
    from oracle.engine import Engine as OEngine, EngineConfig, ScriptedSource
    from synth import SHAPES, gen_requests
    shape = SHAPES["7B"]
    cfg = EngineConfig(block_size=64, num_blocks=1 << 20, T=400, cap=8192, eos_id=1)
    eng = OEngine(cfg, ScriptedSource(1))
    for r in gen_requests(8, shape, 16, 4, 0.5, 8, 8192, 400, eos_id=1, p_range=(64, 1024)):
        eng.admit(r)
    t = time.perf_counter()
    st = eng.step(1 << 20)
    el = time.perf_counter() - t
    return dict(boundaries_per_s=st["windows"] / el, requests_per_s=st["finalized_total"] / el,
                windows=st["windows"], requests=st["finalized_total"], s=el)


def cpu_baseline_legs(timed: int, warmup: int):
    lim, cores, used = _oracle_threads()
    c2 = oracle_c2_slice(timed, warmup)
    med = statistics.median(c2["times"])
    legs = {"c2_slice": {"value": C2["N"] / med, "unit": "branch-tokens/s", "median_step_s": med,
                         "min_step_s": min(c2["times"]), "max_step_s": max(c2["times"]),
                         "prefill_s": c2["prefill_s"], "timed_steps": len(c2["times"])}}
    try:
        legs["c1_full"] = oracle_c1_full()
    except Exception as e:
        legs["c1_full"] = {"failed": repr(e)}
    try:
        legs["control_replay_c3_slice"] = oracle_control_replay()
    except Exception as e:
        legs["control_replay_c3_slice"] = {"failed": repr(e)}
    return dict(value=legs["c2_slice"]["value"], unit="branch-tokens/s", cores=used, kind="oracle",
                sample=f"C2 slice (BASELINE.md §4): 1 request x N={C2['N']} branches, 1.5B shape, fp64 NumPy, "
                       f"P=544, model mode; median of {len(c2['times'])} timed decode steps after the prefill "
                       f"window and {warmup} warm-up steps; weights tiled from one seeded block "
                       f"({c2['gen_s']:.0f}s, untimed)",
                legs=legs, step_s=med)


def run_reference(args, rank, world):
    """The base contract's reference arm: the oracle as it stands, on the host cores, rank 0
    only (other ranks exit without work).  A step = one decode step of the C2 slice."""
    if rank != 0:
        return
    r = cpu_baseline_legs(args.steps, max(1, args.warmup))
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": r["unit"], "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["step_s"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 (BASELINE.json configs[1]) oracle slice: 1 request, N=8, M=4, cap 4096, "
                                   "P=544, 1.5B shape", "step": "one decode step of the slice"},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "legs")},
            "e2e": {"value": r["value"], "unit": r["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def step_roofline(shape, n_avg, attn_bytes_step, ms_step, peaks):
    """Whole decode step against its roofline: t_roofline = sum over kernels of
    max(algorithmic bytes / HBM peak, flops / tensor peak), per decode step at the average
    number of running rows n.  GEMMs: weights once per step + activations in/out; attention:
    the device-counted algorithmic bytes (prefix once per request, suffixes, KV appends);
    RMSNorm: fp32 residual read + bf16 out; sampler: fp32 logits written and read once."""
    bw = peaks.get("hbm_gbs", 6650.0) * 1e9
    tc = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1668.0)) * 1e12
    d, L, V, F = shape.d_model, shape.n_layers, shape.vocab, shape.d_ff
    qkv = shape.qkv_dim
    gemms = {"qkv": (d, qkv, 2), "o": (shape.n_heads * shape.head_dim, d, 4), "gate_up": (d, 2 * F, 2),
             "down": (F, d, 4)}
    per = {}
    for name, (K, N, ob) in gemms.items():
        by = N * K * 2 + n_avg * K * 2 + n_avg * N * ob
        fl = 2.0 * n_avg * N * K
        per[name] = L * max(by / bw, fl / tc)
    by = V * d * 2 + n_avg * d * 2 + n_avg * V * 4
    per["lm_head"] = max(by / bw, 2.0 * n_avg * V * d / tc)
    per["attention"] = attn_bytes_step / bw
    per["rmsnorm"] = (2 * L + 1) * n_avg * d * (4 + 2) / bw
    per["sampler"] = n_avg * V * 4 / bw
    t = sum(per.values())
    return {"t_roofline_ms": t * 1e3, "t_measured_ms": ms_step, "frac": t * 1e3 / ms_step if ms_step > 0 else None,
            "n_avg_running_rows": n_avg, "per_kernel_ms": {k: v * 1e3 for k, v in per.items()},
            "peaks": {"hbm_gbs": bw / 1e9, "bf16_tflops": tc / 1e12,
                      "tc_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernels inside a long step)"},
            "t_measured": "timed region / decode steps (includes admission, prefill and boundaries)"}


# ------------------------------------------------------------------ GPU arm
def relaunch(args) -> int:
    """`bench.py --gpus N` without a torch.distributed environment: start the N ranks here
    (one process per GPU, the driver's own torchrun command line) and pass rank 0's line on."""
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def make_engine(shape, cfg, rank, local, stream, attn_mode):
    from paper_2505_13326_b200 import Engine
    return Engine(shape, "bf16", weight_seed=1234 + rank, block_size=cfg["block_size"], num_blocks=0,
                  max_rows=cfg["concurrent"] * cfg["N"], max_requests=256, max_prompt=cfg["p_range"][1] + 1,
                  T=cfg["T"], cap=cfg["cap"], eos_id=1, temperature=1.0, sampler_seed=7, device=local,
                  stream=stream.cuda_stream, profile=False, attn_mode=attn_mode)


def e2e_leg(shape, cfg, rank, world, local, stream, attn_mode):
    """End to end through the public C-ABI, from an empty engine: sart_admit one C2 batch (64
    requests per GPU) from host buffers, sart_step + sart_collect until every one of them is
    finalized and collected, then the C2 gather of the result records to rank 0 (NCCL).  Wall
    clock on the host around all of it (max over ranks).  H2D / D2H are the bytes the library
    itself copied (sart_profile), i.e. prompts, scripts, admission events and prefill token
    lists up; counter records, finalized records and the selected branches' tokens down."""
    import torch
    import torch.distributed as dist
    from paper_2505_13326_b200 import dist as sdist
    eng = make_engine(shape, cfg, rank, local, stream, attn_mode)
    reqs = make_requests(rank, world, 1 << 20, cfg["concurrent"], shape, cfg)
    want = len(reqs)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eng.reset_profile()
    t0 = time.perf_counter()
    for r in reqs:
        eng.admit(r)
    got, windows, tokens = [], 0, 0
    while len(got) < want:
        st = eng.step(1)
        windows += 1
        got += eng.collect()
        if st["live_rows"] == 0 and st["queued_requests"] == 0 and st["queued_branches"] == 0 and len(got) < want:
            raise RuntimeError("engine idle before every admitted request was collected")
    tokens = st["branch_tokens"]
    recs = sdist.gather_result_records(got, f"cuda:{local}") if world > 1 else None   # C2 (NCCL)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    prof = eng.profile()
    eng.close()
    v = torch.tensor([el, float(tokens), float(len(got)), float(windows), float(prof["h2d_bytes"]),
                      float(prof["d2h_bytes"])], dtype=torch.float64, device="cuda")
    if world > 1:
        mx = v.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
        v[0], v[3] = mx[0], mx[3]
    el_max, tok_all, req_all, win_max, h2d, d2h = (float(x) for x in v)
    if recs is not None and rank == 0:
        assert recs.shape[0] == int(req_all), (recs.shape, req_all)
    return {"value": tok_all / el_max, "unit": "branch-tokens/s", "requests_per_s": req_all / el_max,
            "requests": int(req_all), "windows": int(win_max), "wall_s": el_max,
            "h2d_bytes_per_step": int(h2d / max(1.0, win_max * world)),
            "d2h_bytes_per_step": int(d2h / max(1.0, win_max * world)),
            "step": "one window (per GPU)",
            "includes": "sart_admit of one C2 batch from host buffers (64 requests/GPU, empty engine), every "
                        "window until all are finalized (prefill, decode, boundaries, tail), sart_collect, "
                        + ("NCCL gather of the result records to rank 0" if world > 1 else "no gather (N=1)")}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    import torch
    import torch.distributed as dist
    from synth import SHAPES

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = SHAPES[C2["shape"]]
    cfg = dict(C2)
    cfg["T"] = args.T
    stream = torch.cuda.current_stream()
    eng = make_engine(shape, cfg, rank, local, stream, args.attn_mode)
    windows_needed = args.warmup + args.steps
    # backlog: enough requests that 64 stay resident for every window (~12 finalize per window)
    n_backlog = cfg["concurrent"] + 24 * windows_needed
    reqs = make_requests(rank, world, 0, n_backlog, shape, cfg)
    for r in reqs:
        eng.admit(r)
    counters = torch.zeros(world, 16, dtype=torch.int32, device="cuda")
    mine = torch.zeros(16, dtype=torch.int32, device="cuda")

    def window():
        st = eng.step(1)
        if world > 1:     # C1: all-gather of the admission counters
            dist.all_gather_into_tensor(counters, eng.counters(mine))
        return st

    for _ in range(args.warmup):
        window()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st0 = eng.step(0)
    p0 = eng.profile()
    clk = ClockSampler(local)
    clk.start()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        window()
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1)
    st1 = eng.step(0)
    p1 = eng.profile()
    tokens = st1["branch_tokens"] - st0["branch_tokens"]
    finals = st1["finalized_total"] - st0["finalized_total"]
    dec_steps = st1["steps"] - st0["steps"]
    t = torch.tensor([ms, float(tokens), float(finals), float(dec_steps)], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        t[0] = tmax[0]
    ms_max, tok_all, fin_all = float(t[0]), float(t[1]), float(t[2])
    value = tok_all / (ms_max / 1e3)
    launches = p1["kernel_launches"] - p0["kernel_launches"]

    # ---------------- roofline of the dominant kernel: one more window with per-launch CUDA
    # events around every attention launch (eager launches on the same stream, same workload)
    # window A (profile 2): events before the cascade kernel, between it and the merge, after
    # the merge -> the kernel's own duration; window B (profile 1): no mid event, so the merge
    # keeps its PDL overlap -> the whole operator
    eng.set_profile(2)
    q0 = eng.profile()
    sp0 = eng.step(0)
    eng.step(1)
    torch.cuda.synchronize()
    q1 = eng.profile()
    sp1 = eng.step(0)
    eng.set_profile(1)
    eng.step(1)
    torch.cuda.synchronize()
    q2 = eng.profile()
    eng.set_profile(False)
    stream_ms = q1["attn_stream_ms"] - q0["attn_stream_ms"]       # k_attn_cascade alone (window A)
    attn_bytes = q1["attn_bytes"] - q0["attn_bytes"]
    n_attn = max(1, q1["attn_launches"] - q0["attn_launches"])
    attn_bytes_b = q2["attn_bytes"] - q1["attn_bytes"]            # window B: cascade + merge
    attn_ms_b = q2["attn_ms"] - q1["attn_ms"]
    n_attn_b = max(1, q2["attn_launches"] - q1["attn_launches"])
    peaks = load_peaks()
    try:   # ncu --set full capture of the same kernel in the same workload (tools/attn_traffic.py)
        traffic = json.load(open(os.path.join(ROOT, "profiles", "attn_traffic.json")))
    except Exception:
        traffic = {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    achieved = attn_bytes / (stream_ms / 1e3) / 1e9 if stream_ms > 0 else 0.0
    achieved_m = attn_bytes_b / (attn_ms_b / 1e3) / 1e9 if attn_ms_b > 0 else 0.0
    n_steps_rl = max(1, sp1["steps"] - sp0["steps"])
    roofline = {"bound": "hbm", "kernel": "k_attn_cascade (cascade decode attention, the dominant kernel)",
                "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic.get("dram_bytes_per_launch"),
                "traffic_source": traffic.get("source", "no ncu capture committed (profiles/attn_traffic.json)"),
                "traffic_algorithmic_bytes_at_capture": traffic.get("algorithmic_bytes_per_launch"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s",
                "bytes_per_launch": attn_bytes / n_attn, "launch_avg_ms": stream_ms / n_attn,
                "launches_measured": n_attn,
                "measured_over": "1 eager window after the timed region (%d decode steps), CUDA events on the "
                                 "engine stream before the kernel and between it and the merge" % n_steps_rl,
                "bytes": "algorithmic: prefix KV once per request with a running row + each running suffix "
                         "once + q in / o out (DESIGN.md section 6)",
                # the whole attention operator, merge of the partials included (second kernel)
                "with_merge": {"achieved": achieved_m, "frac": achieved_m / hbm_peak, "launch_avg_ms": attn_ms_b / n_attn_b,
                               "bytes_per_launch": attn_bytes_b / n_attn_b,
                               "measured_over": "the next eager window, events before the cascade and after the merge"},
                "attn_ms_per_step": stream_ms / n_steps_rl}

    # whole decode step vs its roofline; attention bytes per step from the accounted window
    step_rl = step_roofline(shape, tokens / max(1, dec_steps), attn_bytes / max(1, sp1["steps"] - sp0["steps"]),
                            ms_max / max(1, dec_steps), peaks)
    eng.close()

    # ---------------- e2e: the public C-ABI path with host buffers, H2D/D2H inside the timed region
    e2e = None if args.no_e2e else e2e_leg(shape, cfg, rank, world, local, stream, args.attn_mode)
    if world > 1:
        dist.barrier()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            r = cpu_baseline_legs(args.cpu_steps, 2)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample", "legs")}
        except Exception as e:  # never let the baseline kill the bench line
            cpu = {"value": None, "unit": "branch-tokens/s", "cores": len(os.sched_getaffinity(0)),
                   "kind": "oracle", "sample": f"failed: {e!r}"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "branch-tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "C2 (BASELINE.json configs[1]) steady state: 1.5B-shape bf16 random-init, "
                                       "64 concurrent requests/GPU (B=512 rows), N=8, M=4, cap 4096, T=%d, "
                                       "pruning off, prompts U[64,1024], scripted lengths" % cfg["T"],
                           "step": "one window = admission + T decode steps + boundary",
                           "parallelism": f"request-partitioned dp{world}",
                           "l2": "inputs larger than L2 (3.1 GB weights + multi-GB KV per step)"},
                "requests_per_s": fin_all / (ms_max / 1e3), "decode_steps_timed": dec_steps,
                "prefill_ms_timed": p1["prefill_ms"] - p0["prefill_ms"],
                "branch_tokens_timed": tok_all, "gpu_launches": launches, "clocks": clocks,
                "roofline": roofline, "step_roofline": step_rl, "cpu_baseline": cpu, "e2e": e2e}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
