import sys, os, threading, numpy as np
os.environ.setdefault('CUDA_MODULE_LOADING', 'EAGER')
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from gpu_common import gpu_engine
from synth import SHAPES, Request, gen_prompt, gen_weights
shape = SHAPES["small"]
w = gen_weights(shape, "bf16", std=0.02)
eng = [gpu_engine(shape, "bf16", w, tp=(2, r), block_size=16, num_blocks=256, max_rows=16, max_requests=4, max_prompt=64, T=4, cap=16, eos_id=1, enable_forced_tokens=True) for r in range(2)]
ptrs = [e.tp_buffer()[0] for e in eng]
print("bufs", [hex(p) for p in ptrs], flush=True)
for e in eng: e.tp_connect(ptrs=ptrs)
ft = np.full((2, 16), 7, np.int32)
for e in eng: e.admit(Request(0, gen_prompt(1, shape.vocab, 1, 20, 20), 2, 2, -1.0, 0, None), forced_tokens=ft)
import ctypes
def run(e, out, i):
    try: out[i] = e.step(1)
    except Exception as ex: out[i] = repr(ex)
out = [None, None]
ts = [threading.Thread(target=run, args=(eng[i], out, i)) for i in range(2)]
[t.start() for t in ts]; [t.join() for t in ts]
print("step", out, flush=True)
