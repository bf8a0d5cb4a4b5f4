"""DRAM traffic of the cascade attention kernel vs its algorithmic bytes, in the bench workload.

Run under ncu (one GPU):
  ncu --set full --clock-control none -k regex:k_attn_cascade -s <skip> -c <count> \
      --csv --page raw --log-file gpurun_out/attn_full.csv python tools/attn_traffic.py --warm 3
then summarise with
  python tools/attn_traffic.py --summarise gpurun_out/attn_full.csv gpurun_out/attn_traffic_run.log
which writes profiles/attn_traffic.json (read by bench.py for roofline.traffic).

The driven workload is bench.py's C2 (same requests, T=400, B=512); W warm windows run first,
then one window with per-launch accounting (profile=True: eager launches, so ncu sees each
attention launch).  The algorithmic bytes per launch are that window's device-counted
attention bytes / launches (SURVEY §8(d) formula); the captured launches sit mid-window
(-s = W*400*L + 200*L), so the window average matches them to within the suffix growth of
half a window."""
import argparse
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(warm: int, num_blocks: int, config: str = "c2"):
    import bench
    from paper_2505_13326_b200 import Engine
    from synth import SHAPES, gen_requests
    if config == "c5":
        # C5 (BJ configs[4]): 14B, one 8192-token prompt shared by N = 32 branches, M 16,
        # alpha 0.5, beta 16, cap 16384 -- the prefix-heavy case the cascade exists for
        shape = SHAPES["14B"]
        cfg = dict(T=400, cap=16384)
        eng = Engine(shape, "bf16", weight_seed=3, block_size=64, num_blocks=num_blocks, max_rows=64,
                     max_requests=16, max_prompt=8193, T=cfg["T"], cap=cfg["cap"], eos_id=1, temperature=1.0,
                     sampler_seed=5, profile=True)
        reqs = gen_requests(1, shape, 32, 16, 0.5, 16, cfg["cap"], cfg["T"], eos_id=1, p_range=(8193, 8193))
    else:
        cfg = dict(bench.C2)
        shape = SHAPES["1.5B"]
        # a pool that holds all 64 resident requests (R34 needs ~33.3K blocks) but leaves ncu room
        # to back up device memory ON the device between replay passes (a pool sized from all
        # free HBM forces a host-memory backup, under which the replayed run failed to launch)
        eng = Engine(shape, "bf16", weight_seed=1234, block_size=64, num_blocks=num_blocks, max_rows=512,
                     max_requests=256, max_prompt=1025, T=cfg["T"], cap=cfg["cap"], eos_id=1, temperature=1.0,
                     sampler_seed=7, profile=True)   # eager launches (ncu replays single kernels, not graph nodes)
        reqs = bench.make_requests(0, 1, 0, cfg["concurrent"] + 24 * (warm + 2), shape, cfg)
    for r in reqs:
        eng.admit(r)
    eng.step(warm)
    q0 = eng.profile()
    eng.step(1)
    q1 = eng.profile()
    n = q1["attn_launches"] - q0["attn_launches"]
    st = eng.step(0)
    print(json.dumps({"config": config, "attn_bytes": q1["attn_bytes"] - q0["attn_bytes"], "attn_launches": n,
                      "attn_ms": q1["attn_ms"] - q0["attn_ms"], "warm": warm, "live_rows": st["live_rows"],
                      "steps": st["steps"]}), flush=True)
    eng.close()


def summarise(csv_path: str, log_path: str, out_name: str = "attn_traffic.json"):
    rows = list(csv.reader(open(csv_path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    units = rows[hdr_i + 1] if hdr_i + 1 < len(rows) and not rows[hdr_i + 1][0].isdigit() else None
    recs = [dict(zip(hdr, r)) for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0].isdigit()]
    recs = [r for r in recs if re.search("k_attn_cascade", r["Kernel Name"])]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    def val(r, k):
        u = dict(zip(hdr, units)).get(k, "byte") if units else "byte"
        return float(r[k].replace(",", "")) * scale.get(u, 1)
    rd = [val(r, "dram__bytes_read.sum") for r in recs]
    wr = [val(r, "dram__bytes_write.sum") for r in recs]
    log = [json.loads(l) for l in open(log_path) if l.startswith("{")][-1]
    out = {"dram_bytes_per_launch": (sum(rd) + sum(wr)) / len(recs),
           "dram_read_per_launch": sum(rd) / len(recs), "dram_write_per_launch": sum(wr) / len(recs),
           "launches_captured": len(recs),
           "algorithmic_bytes_per_launch": log["attn_bytes"] / log["attn_launches"],
           "source": "ncu, k_attn_cascade mid-window launches of %s window %d (tools/attn_traffic.py)"
                     % (log.get("config", "c2").upper(), log["warm"] + 1)}
    durs = [val(r, "gpu__time_duration.sum") for r in recs if "gpu__time_duration.sum" in r]
    if durs:   # ncu times are serialised and cold-L2: context only
        out["ncu_us_per_launch"] = sum(durs) / len(durs) / 1e3 if max(durs) > 1e4 else sum(durs) / len(durs)
    out["traffic_over_algorithmic"] = out["dram_bytes_per_launch"] / out["algorithmic_bytes_per_launch"]
    json.dump(out, open(os.path.join(ROOT, "profiles", out_name), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--summarise", nargs=2)
    ap.add_argument("--num-blocks", type=int, default=40000)
    ap.add_argument("--config", default="c2", choices=["c2", "c5"])
    ap.add_argument("--out", default="attn_traffic.json")
    a = ap.parse_args()
    if a.summarise:
        summarise(*a.summarise, a.out)
    else:
        run(a.warm, a.num_blocks, a.config)
