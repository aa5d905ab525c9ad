"""Plain-numpy restatement of the reference ``redve`` hot path (TEST ORACLE).

Test infrastructure only (see ``oracle/__init__.py``).  Single image, fp64,
single-threaded, exactly the reference's arithmetic order where it matters
for decisions (FFT-based operators, MGS QR with two re-orthogonalisation
passes, scipy-``cg`` recursion).  Paths below are relative to
``/root/reference/pkg/src/redve/``.
"""

from __future__ import annotations

import math
import time

import numpy as np
from scipy.linalg import solve_triangular

# ---------------------------------------------------------------------------
# PSFs and circulant operators                           (imaging.py:46-204)
# ---------------------------------------------------------------------------


def psf_taps(kind: str, size: int, std: float | None = None) -> np.ndarray:
    """imaging.py:71-92 -- normalised uniform / Gaussian k x k kernel."""
    if size < 1 or size % 2 == 0:
        raise ValueError("odd size >= 1 required")
    if kind == "uniform":
        return np.full((size, size), 1.0 / size**2)
    if kind != "gaussian" or std is None or std <= 0:
        raise ValueError("bad psf")
    r = size // 2
    g = np.arange(-r, r + 1, dtype=np.float64)
    a, b = np.meshgrid(g, g, indexing="ij")
    t = np.exp(-(a**2 + b**2) / (2.0 * std**2))
    return t / t.sum()


def transfer_function(taps: np.ndarray, shape) -> np.ndarray:
    """imaging.py:113-129 -- DFT of the kernel embedded with its centre at (0,0)."""
    k = taps.shape[0]
    r = k // 2
    emb = np.zeros(shape)
    emb[:k, :k] = taps
    return np.fft.fft2(np.roll(emb, (-r, -r), axis=(0, 1)))


def fft_conv(x: np.ndarray, spec: np.ndarray) -> np.ndarray:
    """imaging.py:132-139 -- circular convolution through the DFT (real part)."""
    return np.fft.ifft2(np.fft.fft2(x) * spec).real


class CirculantBlur:
    """imaging.py:147-170 (``Blur``): H x = k * x, H^T z = correlation."""

    is_circulant = True

    def __init__(self, taps: np.ndarray, shape):
        self.taps = np.asarray(taps, dtype=np.float64)
        self.in_shape = self.out_shape = tuple(shape)
        self.spectrum = transfer_function(self.taps, self.in_shape)

    def apply(self, x):
        return fft_conv(x, self.spectrum)

    def adjoint(self, z):
        return fft_conv(z, np.conj(self.spectrum))


class BlurDecimate:
    """imaging.py:173-204 (``BlurDownsample``): keep indices == 0 mod s."""

    is_circulant = False

    def __init__(self, taps: np.ndarray, factor: int, shape):
        self.taps = np.asarray(taps, dtype=np.float64)
        self.factor = int(factor)
        self.in_shape = tuple(shape)
        h, w = shape
        self.out_shape = ((h + factor - 1) // factor, (w + factor - 1) // factor)
        self.spectrum = transfer_function(self.taps, self.in_shape)

    def apply(self, x):
        s = self.factor
        return fft_conv(x, self.spectrum)[::s, ::s]

    def adjoint(self, z):
        s = self.factor
        up = np.zeros(self.in_shape)
        up[::s, ::s] = z
        return fft_conv(up, np.conj(self.spectrum))


def noise_field(shape, sigma: float, seed: int) -> np.ndarray:
    """imaging.py:207-218 -- PCG64 + Box-Muller, bit-identical to the reference."""
    gen = np.random.Generator(np.random.PCG64(seed))
    n = int(np.prod(shape))
    u1 = 1.0 - gen.random(n)
    u2 = gen.random(n)
    return sigma * (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).reshape(shape)


def measure(truth, op, sigma: float, seed: int):
    """imaging.py:221-231 (``degrade``)."""
    clean = op.apply(np.asarray(truth, dtype=np.float64))
    return clean if sigma == 0 else clean + noise_field(clean.shape, sigma, seed)


def psnr(x, ref) -> float:
    """imaging.py:234-248 -- fixed peak 255; +inf identical, -inf overflow."""
    mse = np.mean((np.asarray(x, np.float64) - np.asarray(ref, np.float64)) ** 2)
    if mse == 0.0:
        return math.inf
    if not np.isfinite(mse):
        return -math.inf
    return 10.0 * np.log10(255.0**2 / mse)


def scene(height: int, width: int | None = None) -> np.ndarray:
    """imaging.py:251-270 (``synthetic_image``) -- disk, square, stripes."""
    width = height if width is None else width
    ii, jj = np.meshgrid(np.arange(height), np.arange(width), indexing="ij")
    v = ii / max(height - 1, 1)
    u = jj / max(width - 1, 1)
    img = 110.0 + 60.0 * np.sin(2 * np.pi * (1.5 * u + 0.5)) * np.cos(2 * np.pi * v)
    img[((u - 0.3) ** 2 + (v - 0.35) ** 2) < 0.04] = 220.0
    sq = (np.abs(u - 0.72) < 0.12) & (np.abs(v - 0.68) < 0.12)
    img[sq] = 35.0
    band = (np.abs(u + v - 1.35) < 0.18) & ~sq
    img[band] += 45.0 * np.sin(24 * np.pi * (u - v))[band]
    return np.clip(img, 5.0, 250.0)


# ---------------------------------------------------------------------------
# Denoisers                                               (denoisers.py:21-129)
# ---------------------------------------------------------------------------


def identity(x):
    """denoisers.py:21-27."""
    return np.array(x, dtype=np.float64, copy=True)


def gaussian_filter(x, std: float = 0.55, support: int = 5):
    """denoisers.py:30-46 -- FFT circular convolution, spectrum rebuilt per call."""
    x = np.asarray(x, dtype=np.float64)
    return fft_conv(x, transfer_function(psf_taps("gaussian", support, std), x.shape))


def patch_weight_maps(x, patch_radius=1, search_radius=3, h=110.0, balance_iters=20):
    """denoisers.py:83-111 -- raw exp(-d^2/h^2) maps + symmetric balancing."""
    x = np.asarray(x, dtype=np.float64)
    box = transfer_function(psf_taps("uniform", 2 * patch_radius + 1), x.shape)
    inv_h2 = 1.0 / h**2
    offs, maps = [], []
    rng = range(-search_radius, search_radius + 1)
    for di in rng:
        for dj in rng:
            diff2 = (x - np.roll(x, (-di, -dj), axis=(0, 1))) ** 2
            d2 = fft_conv(diff2, box)
            offs.append((di, dj))
            maps.append(np.exp(-np.maximum(d2, 0.0) * inv_h2))
    for _ in range(balance_iters):
        s = np.zeros_like(x)
        for w in maps:
            s += w
        g = 1.0 / np.sqrt(s)
        maps = [w * g * np.roll(g, (-di, -dj), axis=(0, 1)) for (di, dj), w in zip(offs, maps)]
    return offs, maps


def apply_weight_maps(offs, maps, z):
    """denoisers.py:113-119."""
    out = np.zeros_like(z, dtype=np.float64)
    for (di, dj), w in zip(offs, maps):
        out += w * np.roll(z, (-di, -dj), axis=(0, 1))
    return out


def patch_weighted(x, patch_radius=1, search_radius=3, h=110.0, balance_iters=20):
    """denoisers.py:126-129."""
    x = np.asarray(x, dtype=np.float64)
    offs, maps = patch_weight_maps(x, patch_radius, search_radius, h, balance_iters)
    return apply_weight_maps(offs, maps, x)


# ---------------------------------------------------------------------------
# RED objective and its fixed-point step                  (objective.py:44-135)
# ---------------------------------------------------------------------------

CG_RTOL, CG_MAXITER, CG_ABORT = 1e-6, 200, 1e-4  # objective.py:35-37


class CgFailed(ArithmeticError):
    pass


def scipy_cg(matvec, b, x0, rtol=CG_RTOL, maxiter=CG_MAXITER):
    """Restatement of scipy 1.18.1 ``cg`` (sparse/linalg/_isolve/iterative.py:
    311-430) with M = I and atol = 0: stop when ||r|| < rtol*||b||, tested
    *before* every iteration (so a warm start may return x0 unchanged);
    residual updated recursively.  Returns (x, info, iterations)."""
    bn = np.linalg.norm(b)
    atol = max(0.0, rtol * float(bn))
    if bn == 0:
        return b, 0, 0
    x = np.array(x0, dtype=np.float64, copy=True)
    r = b - matvec(x) if x.any() else b.copy()
    rho_old = None
    p = None
    for it in range(maxiter):
        if np.linalg.norm(r) < atol:
            return x, 0, it
        rho = np.dot(r, r)
        if it > 0:
            p *= rho / rho_old
            p += r
        else:
            p = r.copy()
        q = matvec(p)
        a = rho / np.dot(p, q)
        x += a * p
        r -= a * q
        rho_old = rho
    return x, maxiter, maxiter


class Red:
    """objective.py:44-121 (``RedObjective``)."""

    def __init__(self, op, y, sigma, alpha, denoiser):
        if sigma <= 0 or alpha <= 0:
            raise ValueError("sigma, alpha must be > 0")
        self.op, self.sigma, self.alpha, self.denoiser = op, float(sigma), float(alpha), denoiser
        self.y = np.asarray(y, dtype=np.float64)
        self.hty = op.adjoint(self.y) / self.sigma**2                        # :70
        self.denom = (np.abs(op.spectrum) ** 2 / self.sigma**2 + self.alpha  # :71-72
                      if op.is_circulant else None)
        self.cg_iters = []

    def data_fidelity(self, x):                                              # :78-81
        r = self.op.apply(x) - self.y
        return float(np.vdot(r, r).real) / (2.0 * self.sigma**2)

    def regularizer(self, x):                                                # :83-85
        return 0.5 * float(np.vdot(x, x - self.denoiser(x)).real)

    def cost(self, x):                                                       # :87-88
        return self.data_fidelity(x) + self.alpha * self.regularizer(x)

    def gradient(self, x):                                                   # :90-93
        d = self.op.adjoint(self.op.apply(x) - self.y) / self.sigma**2
        return d + self.alpha * (x - self.denoiser(x))

    def normal_matvec(self, v):                                              # :97-98
        return self.op.adjoint(self.op.apply(v)) / self.sigma**2 + self.alpha * v

    def fp_step(self, x):                                                    # :100-121
        x = np.asarray(x, dtype=np.float64)
        rhs = self.hty + self.alpha * self.denoiser(x)
        if self.denom is not None:
            return np.fft.ifft2(np.fft.fft2(rhs) / self.denom).real
        shape = self.op.in_shape
        mv = lambda v: self.normal_matvec(v.reshape(shape)).ravel()
        sol, info, its = scipy_cg(mv, rhs.ravel(), x.ravel())
        self.cg_iters.append(its)
        sol = sol.reshape(shape)
        if info != 0:
            res = np.linalg.norm(self.normal_matvec(sol) - rhs)
            if res > CG_ABORT * np.linalg.norm(rhs):
                raise CgFailed(f"cg residual {res:.3e}")
        return sol


# ---------------------------------------------------------------------------
# Vector extrapolation                                 (extrapolation.py:154-386)
# ---------------------------------------------------------------------------


class VeStationary(Exception):
    pass


def mgs(u, tol=1e-12):
    """extrapolation.py:159-196 -- MGS, two projection sweeps per column,
    relative rank cut r_ii < tol*r_11.  Returns (Q, R, rank)."""
    u = np.asarray(u, dtype=np.float64)
    n, k = u.shape
    q = np.zeros((n, k))
    r = np.zeros((k, k))
    rank, r11 = k, 0.0
    for i in range(k):
        v = u[:, i].copy()
        for _sweep in range(2):
            for j in range(i):
                c = q[:, j] @ v
                r[j, i] += c
                v -= c * q[:, j]
        d = float(np.linalg.norm(v))
        r[i, i] = d
        if i == 0:
            if d < 1e-300:
                raise VeStationary()
            r11 = d
        elif d < tol * r11:
            rank = i
            break
        q[:, i] = v / d
    return q, r, rank


def _annihilate(r, order):
    """extrapolation.py:241-254 -- order-e MPE-form weights; None if degenerate."""
    cp = solve_triangular(r[:order, :order], -r[:order, order], lower=False)
    c = np.append(cp, 1.0)
    s = float(c.sum())
    if abs(s) < 1e-12 * float(np.abs(c).sum()) or not np.isfinite(s):
        return None
    return c, c / s


def weights_rre(r):
    """extrapolation.py:263-273."""
    one = np.ones(r.shape[0])
    d = solve_triangular(r, solve_triangular(r, one, trans="T", lower=False), lower=False)
    return d, d / float(d.sum())


def weights_svdmpe(r):
    """extrapolation.py:199-214, 276-284; None if the singular vector sums to ~0."""
    try:
        _, _, vt = np.linalg.svd(r)
    except np.linalg.LinAlgError:
        return None
    v = vt[-1].copy()
    s = float(v.sum())
    if abs(s) < 1e-12 or not np.isfinite(s):
        return None
    return v, v / s


def extrapolate(rows, method="mpe", tol=1e-12):
    """extrapolation.py:319-386 (``extrapolate_once``) on an array of kappa+2
    iterate rows.  Returns dict(vector, converged, extrapolated, kappa_used,
    method, fallback_from, c, gamma, stability_sum)."""
    rows = np.asarray(rows, dtype=np.float64)
    kappa = rows.shape[0] - 2
    out = dict(converged=False, extrapolated=False, kappa_used=0, method=None,
               fallback_from=None, c=None, gamma=None, stability_sum=None)
    u = np.diff(rows, axis=0).T                                              # :154-156
    try:
        q, r, e = mgs(u, tol)
    except VeStationary:
        out.update(vector=rows[0].copy(), converged=True)
        return out
    if not (np.all(np.isfinite(r)) and np.all(np.isfinite(q))):            # :350-358
        out.update(vector=rows[-1].copy())
        return out
    if e == kappa + 1:
        w, used = None, method
        if method == "mpe":
            w = _annihilate(r, kappa)
        elif method == "svdmpe":
            w = weights_svdmpe(r)
        if method == "rre" or w is None:
            if method != "rre":
                out["fallback_from"] = method
            w, used = weights_rre(r), "rre"
        c, g = w
        k_eff, qq, rr, base = kappa, q, r, rows[0]
    else:
        w = _annihilate(r, e)
        if w is None:
            out.update(vector=rows[-1].copy())
            return out
        c, g = w
        used = method
        k_eff, qq, rr, base = e, q[:, : e + 1], r[: e + 1, : e + 1], rows[0]
    xi = 1.0 - np.cumsum(g[:k_eff])                                          # :295-305
    eta = rr[:k_eff, :k_eff] @ xi
    vec = base + qq[:, :k_eff] @ eta                                         # :308-316
    out.update(vector=vec, extrapolated=True, kappa_used=k_eff, method=used, c=c,
               gamma=g, stability_sum=float(np.abs(g).sum()))
    return out


# ---------------------------------------------------------------------------
# Drivers                                                   (solvers.py:206-385)
# ---------------------------------------------------------------------------

DENSE_LOG_LIMIT = 128 * 128  # solvers.py:34


class NonFinite(ArithmeticError):
    def __init__(self, msg, trace):
        super().__init__(msg)
        self.trace = trace


class Trace:
    """solvers.py:51-95 -- one record per baseline-map evaluation."""

    def __init__(self):
        self.iters, self.cost, self.psnr, self.step_norm, self.gamma = [], [], [], [], []
        self.cycles = []  # extrapolation dicts of accepted cycles
        self.elapsed = []

    def first_iter_at_cost(self, thr):
        for k, c in zip(self.iters, self.cost):
            if c is not None and c <= thr:
                return k
        return None

    def as_arrays(self):
        nan = lambda v: np.nan if v is None else v
        return dict(
            iter=np.array(self.iters, dtype=np.int64),
            cost=np.array([nan(c) for c in self.cost]),
            psnr=np.array([nan(p) for p in self.psnr]),
            step_norm=np.array(self.step_norm),
            gamma_abs_sum=np.array([nan(g) for g in self.gamma]),
        )


class _Rec:
    """solvers.py:206-262 (``_Recorder``)."""

    def __init__(self, n, step, objective, reference, tol, budget, track_best):
        self.objective, self.reference = objective, reference
        self.tol, self.budget = tol, budget
        self.trace = Trace()
        self.k = 0
        self.every = 1 if n <= DENSE_LOG_LIMIT else 5
        self.track = track_best and objective is not None
        self.best_cost, self.best_x = math.inf, None
        self.t0 = time.perf_counter()

    def initial(self, x0):
        if self.track:
            c = float(self.objective(x0))
            if np.isfinite(c):
                self.best_cost, self.best_x = c, x0.copy()

    def record(self, xp, xn):
        """Returns 'converged' / 'budget' / None (continue)."""
        self.k += 1
        den = float(np.linalg.norm(xp)) or 1.0
        sn = float(np.linalg.norm(xn - xp)) / den
        cost = ps = None
        cad = self.k % self.every == 0
        if cad and self.objective is not None:
            cost = float(self.objective(xn))
            if self.track and cost < self.best_cost:
                self.best_cost, self.best_x = cost, xn.copy()
        if cad and self.reference is not None:
            ps = psnr(xn, self.reference)
        t = self.trace
        t.iters.append(self.k)
        t.cost.append(cost)
        t.psnr.append(ps)
        t.step_norm.append(sn)
        t.gamma.append(None)
        t.elapsed.append(time.perf_counter() - self.t0)
        if not np.all(np.isfinite(xn)):
            raise NonFinite(f"iterate diverged at inner step {self.k}", t)
        if cost is not None and not np.isfinite(cost):
            raise NonFinite(f"objective diverged at inner step {self.k}", t)
        if sn <= self.tol:                                                   # :98-107
            return "converged"
        if self.k >= self.budget:
            return "budget"
        return None

    def finalize(self, x):
        if not self.track or self.best_x is None:
            return x
        c = float(self.objective(x))
        if np.isfinite(c) and c <= self.best_cost:
            return x
        return self.best_x


def run_fp(step, x0, budget, tol=0.0, objective=None, reference=None):
    """solvers.py:288-298 (``run_fixed_point``) on flat vectors."""
    x = np.array(x0, dtype=np.float64, copy=True).ravel()
    rec = _Rec(x.size, step, objective, reference, tol, budget, False)
    while True:
        xn = step(x)
        d = rec.record(x, xn)
        x = xn
        if d is not None:
            return x, rec.trace


def run_cycling(step, x0, budget, method="mpe", m=0, kappa=5, tol=0.0, objective=None,
                reference=None, stabilization=0, rank_tol=1e-12):
    """solvers.py:340-385 (``run_ve_cycling``) on flat vectors."""
    x = np.array(x0, dtype=np.float64, copy=True).ravel()
    rec = _Rec(x.size, step, objective, reference, tol, budget, True)
    rec.initial(x)
    clen = m + kappa + 1
    while True:
        xs = [x]
        conv = False
        for _ in range(clen):
            xn = step(x)
            d = rec.record(x, xn)
            x = xn
            xs.append(x)
            if d == "converged":
                conv = True
                break
            if d == "budget":
                break
        if conv:
            break
        if len(xs) == clen + 1:
            res = extrapolate(np.asarray(xs[m:]), method, rank_tol)
            if res["converged"]:
                x = res["vector"]
                break
            if res["extrapolated"] and np.all(np.isfinite(res["vector"])):
                x = res["vector"]
                rec.trace.gamma[-1] = res["stability_sum"]
                rec.trace.cycles.append(res)
        if rec.k >= budget:
            break
    for _ in range(stabilization):
        xn = step(x)
        rec.record(x, xn)
        x = xn
    return rec.finalize(x), rec.trace


def red_problem(red: Red):
    """objective.py:124-135 (``as_fixed_point_problem``): flat step + cost."""
    shape = red.op.in_shape
    step = lambda v: red.fp_step(v.reshape(shape)).ravel()
    cost = lambda v: red.cost(v.reshape(shape))
    return step, cost
