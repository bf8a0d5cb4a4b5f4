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
import threading
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


def request_bytes(r):
    b = r.prompt.nbytes
    if r.script is not None:
        b += r.script.forced_len.nbytes + r.script.scores.nbytes + r.script.final_score.nbytes + r.script.answer.nbytes
    return b


# ------------------------------------------------------------------ oracle (CPU) arm
def oracle_sample(steps: int, warmup: int, T: int):
    """The oracle as it stands (fp64 numpy) on a bounded C2 sample: 1 request with N=8
    branches (1.5B shape, P=64 prompt, scripted lengths), timed per decode step."""
    import numpy as np
    from oracle.engine import Engine as OEngine, EngineConfig, ModelSource
    from oracle.model import Model
    from synth import SHAPES, gen_requests
    shape = SHAPES[C2["shape"]]
    t0 = time.time()
    # timing input only: plain fp32 normals (the values do not change the oracle's cost)
    rng = np.random.default_rng(0)
    w = {}
    from synth import weight_names, weight_shapes
    shp = weight_shapes(shape)
    for name in weight_names(shape):
        w[name] = (rng.standard_normal(shp[name], dtype=np.float32) * 0.02).astype(np.float32)
        if name.endswith("norm"):
            w[name] += 1.0
    gen_s = time.time() - t0
    cfg = EngineConfig(block_size=64, num_blocks=4096, T=1, cap=C2["cap"], eos_id=1)
    eng = OEngine(cfg, ModelSource(Model(shape, w), cfg, prm_scores=False))
    req = gen_requests(1, shape, C2["N"], C2["M"], C2["alpha"], C2["beta"], C2["cap"], T, eos_id=1,
                       p_range=(64, 64))[0]
    eng.admit(req)
    times = []
    for i in range(warmup + steps):
        t = time.perf_counter()
        eng.step(1)
        dt = time.perf_counter() - t
        if i >= warmup:
            times.append(dt)
    cores = len(os.sched_getaffinity(0))
    per_step = sum(times) / len(times)
    return dict(value=C2["N"] / per_step, unit="branch-tokens/s", cores=cores, kind="oracle",
                sample=f"1 request x N={C2['N']} branches, 1.5B shape fp64 numpy, P=64, {steps} timed decode "
                       f"steps after {warmup} warm-up (first includes prefill); weight gen {gen_s:.0f}s untimed",
                step_s=per_step)


def run_reference(args, rank, world):
    if rank != 0:
        return
    r = oracle_sample(args.steps, max(1, args.warmup), args.T)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": r["unit"], "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["step_s"] * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2 oracle sample (BASELINE.json configs[1])", "shape": "1.5B",
                       "branches": C2["N"], "M": C2["M"], "cap": C2["cap"]},
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
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
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = SHAPES[C2["shape"]]
    cfg = dict(C2)
    cfg["T"] = args.T
    stream = torch.cuda.current_stream()
    eng = Engine(shape, "bf16", weight_seed=1234 + rank, block_size=cfg["block_size"], num_blocks=0,
                 max_rows=cfg["concurrent"] * cfg["N"], max_requests=256, max_prompt=cfg["p_range"][1] + 1,
                 T=cfg["T"], cap=cfg["cap"], eos_id=1, temperature=1.0, sampler_seed=7, device=local,
                 stream=stream.cuda_stream, profile=False, attn_mode=args.attn_mode)
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
            eng.export_counters(mine.data_ptr())
            dist.all_gather_into_tensor(counters, mine)
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
    eng.set_profile(True)
    q0 = eng.profile()
    sp0 = eng.step(0)
    eng.step(1)
    torch.cuda.synchronize()
    q1 = eng.profile()
    sp1 = eng.step(0)
    eng.set_profile(False)
    attn_ms = q1["attn_ms"] - q0["attn_ms"]
    attn_bytes = q1["attn_bytes"] - q0["attn_bytes"]
    n_attn = max(1, q1["attn_launches"] - q0["attn_launches"])
    peaks = load_peaks()
    try:   # ncu --set full capture of the same kernel in the same workload (tools/attn_traffic.py)
        traffic = json.load(open(os.path.join(ROOT, "profiles", "attn_traffic.json")))
    except Exception:
        traffic = {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    achieved = attn_bytes / (attn_ms / 1e3) / 1e9 if attn_ms > 0 else 0.0
    roofline = {"bound": "hbm", "kernel": "k_attn_cascade + k_attn_merge (cascade decode attention)",
                "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic.get("dram_bytes_per_launch"),
                "traffic_source": traffic.get("source", "no ncu capture committed (profiles/attn_traffic.json)"),
                "traffic_algorithmic_bytes_at_capture": traffic.get("algorithmic_bytes_per_launch"),
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s",
                "bytes_per_launch": attn_bytes / n_attn, "launch_avg_ms": attn_ms / n_attn,
                "launches_measured": n_attn,
                "measured_over": "1 eager window after the timed region (%d decode steps)" % (sp1["steps"] - sp0["steps"]),
                "attn_ms_per_step": attn_ms / max(1, sp1["steps"] - sp0["steps"])}

    # whole decode step vs its roofline; attention bytes per step from the accounted window
    step_rl = step_roofline(shape, tokens / max(1, dec_steps), attn_bytes / max(1, sp1["steps"] - sp0["steps"]),
                            ms_max / max(1, dec_steps), peaks)

    # ---------------- e2e: the public C-ABI path with host buffers, H2D/D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        extra = make_requests(rank, world, n_backlog + 1000, cfg["concurrent"], shape, cfg)
        h2d = sum(request_bytes(r) for r in extra)
        d2h = 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_tok0 = eng.step(0)["branch_tokens"]
        for r in extra:
            eng.admit(r)
        for _ in range(args.steps):
            eng.step(1)
            res = eng.collect()
            d2h += sum(192 + 4 * len(x["tokens"]) for x in res)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        e_tok = eng.step(0)["branch_tokens"] - e_tok0
        e2e_v = torch.tensor([el, float(e_tok)], dtype=torch.float64, device="cuda")
        if world > 1:
            mx = e2e_v.clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            dist.all_reduce(e2e_v, op=dist.ReduceOp.SUM)
            e2e_v[0] = mx[0]
        e2e = {"value": float(e2e_v[1]) / float(e2e_v[0]), "unit": "branch-tokens/s",
               "windows": args.steps,
               "h2d_bytes_per_step": h2d // max(1, args.steps), "d2h_bytes_per_step": d2h // max(1, args.steps),
               "includes": "admit (host prompts/scripts), prefill, decode windows, collect (D2H records+tokens)"}
    # C2: gather of result records to rank 0 (counts only here)
    if world > 1:
        dist.barrier()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            r = oracle_sample(2, 1, cfg["T"])
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
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
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
