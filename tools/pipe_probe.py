import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1805_02158_b200 as rv
from paper_1805_02158_b200 import pipeline as pl, batch as bt
from paper_1805_02158_b200.synth import voronoi_scene
B, n = 64, 256
op = rv.Blur(rv.make_psf("uniform", 9), (n, n))
truths = np.stack([voronoi_scene(s, n) for s in range(B)])
clean = np.asarray(op.apply(truths))
ys = np.stack([clean[i] + rv.gaussian_noise((n, n), float(np.sqrt(2)), i) for i in range(B)])
cfg = rv.SolveConfig(method="fp-ve", ve_method="mpe", m=0, kappa=5, max_inner_steps=200)
yh = torch.from_numpy(ys).pin_memory()
den = rv.Median3()
T = []
oRB, osb = pl.RedBatch, pl.solve_batch
def RB(*a, **k):
    t = time.perf_counter(); r = oRB(*a, **k); T.append(("create", time.perf_counter() - t)); return r
def SB(b, x0, c):
    t = time.perf_counter(); res = b.solve(x0, c); t1 = time.perf_counter()
    trs = [res.trace(i) for i in range(b.B)]; t2 = time.perf_counter()
    T.append(("solve", t1 - t)); T.append(("traces", t2 - t1)); return res.x, trs
pl.RedBatch, pl.solve_batch = RB, SB
for rep in range(2):
    T.clear()
    t0 = time.perf_counter()
    k = 0
    for xh, trs in rv.solve_stream(op, (yh for _ in range(10)), float(np.sqrt(2)), 0.02, den, cfg):
        k += 1
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    print("total per step ms", 1e3 * tot / 10)
    for name in ("create", "solve", "traces"):
        v = [1e3 * t for n_, t in T if n_ == name]
        print(name, [round(x, 2) for x in v])
# device-only repeated solve
b = rv.RedBatch(op, yh, float(np.sqrt(2)), 0.02, den)
yd = b.y
for _ in range(3): b.solve(yd, cfg)
t = time.perf_counter()
for _ in range(5): b.solve(yd, cfg)
print("repeat solve ms", 1e3 * (time.perf_counter() - t) / 5)
