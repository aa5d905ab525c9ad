"""Does running two half-batches concurrently (two contexts / streams, two
host threads) beat one full batch?  configs[1] shapes.

python tools/concurrency_probe.py [B] [reps]"""
import ctypes as C
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1805_02158_b200 as rv
from paper_1805_02158_b200 import _native as nat
from paper_1805_02158_b200.synth import voronoi_scene

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = 256
op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
truths = np.stack([voronoi_scene(s, n) for s in range(B)])
clean = np.asarray(op.apply(truths))
ys = np.stack([clean[i] + rv.gaussian_noise((n, n), float(np.sqrt(2)), i) for i in range(B)])
cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", m=0, kappa=5, max_inner_steps=200)
yd = torch.from_numpy(ys).cuda()

full = rv.RedBatch(op, yd, float(np.sqrt(2)), 0.02, rv.Median3())
for _ in range(2):
    full.solve(yd, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    full.solve(yd, cfg)
torch.cuda.synchronize()
t_full = (time.perf_counter() - t0) / reps
print(f"one batch of {B}: {t_full * 1e3:.2f} ms/solve-step")

lib = nat.library()
halves = []
for k in range(2):
    h = C.c_void_p()
    assert lib.redve_create(C.byref(h), 0) == 0
    st = torch.cuda.Stream()
    lib.redve_set_stream(h, C.c_void_p(st.cuda_stream))
    key = (0, threading.get_ident())
    saved = nat._ctx.get(key)
    nat._ctx[key] = h
    with torch.cuda.stream(st):
        yb = yd[k * B // 2:(k + 1) * B // 2].clone()
        bt = rv.RedBatch(op, yb, float(np.sqrt(2)), 0.02, rv.Median3())
        for _ in range(2):
            bt.solve(yb, cfg)
    nat._ctx[key] = saved
    st.synchronize()
    halves.append((h, st, yb, bt))


def run(k, out):
    h, st, yb, bt = halves[k]
    with torch.cuda.stream(st):
        for _ in range(reps):
            bt.solve(yb, cfg)
    st.synchronize()


torch.cuda.synchronize()
t0 = time.perf_counter()
ths = [threading.Thread(target=run, args=(k, None)) for k in range(2)]
for t in ths:
    t.start()
for t in ths:
    t.join()
t_conc = (time.perf_counter() - t0) / reps
print(f"two concurrent halves of {B // 2}: {t_conc * 1e3:.2f} ms/solve-step "
      f"(speed-up {t_full / t_conc:.3f})")
