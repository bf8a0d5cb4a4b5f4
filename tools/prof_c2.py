"""Drive the C2 bench workload to a mid-job state, then run a profiled slice.

usage: python tools/prof_c2.py [--warm W] [--steps S]
Runs W full windows (T=400) to grow the suffixes, then S more windows.  Meant to run
under ncu with -s/-c selecting launches of the last window."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2505_13326_b200 import Engine  # noqa: E402
from synth import SHAPES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--warm", type=int, default=3)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--T", type=int, default=400)
ap.add_argument("--num-blocks", type=int, default=0, help="0: pool from free HBM (use ~40000 under ncu --set full)")
a = ap.parse_args()
cfg = dict(bench.C2)
cfg["T"] = a.T
shape = SHAPES["1.5B"]
eng = Engine(shape, "bf16", weight_seed=1, block_size=64, num_blocks=a.num_blocks, max_rows=512, max_requests=256,
             max_prompt=1025, T=cfg["T"], cap=cfg["cap"], eos_id=1, profile=True)
for r in bench.make_requests(0, 1, 0, 200, shape, cfg):
    eng.admit(r)
t = time.time()
st = eng.step(a.warm)
print("warm", st, time.time() - t, flush=True)
t = time.time()
st = eng.step(a.steps)
print("run", st, time.time() - t, eng.profile(), flush=True)
