// Gradient-step baselines (solvers.py:274-337): one kernel per step evaluates
// grad E(v) = H^T H v / sigma^2 + alpha v - H^T y / sigma^2 - alpha f(v)
// (objective.py:90-93 regrouped: H^T y / sigma^2 is the problem's precomputed
// right-hand side) and takes the step, with the recorder's step-norm sums and
// the last-CTA record fused in.
//
// Circulant H (Blur): H^T H is the periodic convolution with the PSF's
// autocorrelation a(d) = sum_i h(i) h(i + d), radius R = ksize - 1; for a rank-
// one PSF a is rank one too, so the stencil is two 1-D passes over a shared
// tile (17 + 17 taps per pixel for the 9x9 box instead of two FFT round trips).
// BlurDownsample: A v comes from the fused normal operator (sr.cu, CG_PLAIN)
// and this kernel is the elementwise epilogue.
#include "denoise.cuh"
#include "grad.cuh"

namespace redve {

namespace {

constexpr int GT_H = 16, GT_W = 64, GT_THREADS = 256;

inline int cdivg(long long a, long long b) { return (int)((a + b - 1) / b); }

int ew_chunks(long long N) {
  int c = cdivg(N, GT_THREADS * 8);
  return c > 64 ? 64 : (c < 1 ? 1 : c);
}

struct Acc {
  double d2 = 0.0, x2 = 0.0, nf = 0.0;
};

// x_{k+1} (and y_{k+1}) at one pixel; returns nothing, accumulates the sums.
__device__ __forceinline__ void grad_update(const GradArgs& a, int b, long long i, double vv,
                                            double hh, double* xo, const double* xp, Acc& acc) {
  const long long o = (long long)b * a.H * a.W + i;
  const double g = fma(a.alpha, vv - a.f[o], hh) - a.hty[o];
  if (a.gout) {  // RedObjective.gradient: grad E(v) itself, no step
    a.gout[o] = g;
    return;
  }
  const double xn = fma(-a.step, g, vv);
  xo[i] = xn;
  const double xprev = a.ynext ? xp[i] : vv;
  if (a.ynext) a.ynext[o] = fma(a.beta, xn - xprev, xn);
  const double d = xn - xprev;
  acc.d2 = fma(d, d, acc.d2);
  acc.x2 = fma(xprev, xprev, acc.x2);
  acc.nf += isfinite(xn) ? 0.0 : 1.0;
}

__device__ __forceinline__ void grad_finish(const GradArgs& a, int b, Acc acc, int nblk, int blk) {
  if (a.gout) return;
  __shared__ double red[96];
  double v[3] = {acc.d2, acc.x2, acc.nf};
  block_sum<3>(v, red);
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) a.partials[((long long)b * nblk + blk) * 3 + q] = v[q];
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double t[3];
  if (lastb) gather_partials<3>(a.partials + (long long)b * nblk * 3, nblk, t, red);
  if (lastb && threadIdx.x == 0) record_step(a.st[b], b, t[0], t[1], t[2], a.S, a.ctl, a.tr);
}

}  // namespace

// Circulant route: v tile + R halo in shared memory, separable or full stencil.
__global__ void __launch_bounds__(GT_THREADS) k_grad_stencil(GradArgs a) {
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.ctl.phase)) return;
  extern __shared__ double sm[];
  const int R = a.R, H = a.H, W = a.W, T = 2 * R + 1;
  const int TWX = GT_W + 2 * R, THX = GT_H + 2 * R;
  const bool sep = a.au != nullptr;
  double* taps = sm;                        // sep: [av | au]; full: T*T
  const int ntaps = sep ? 2 * T : T * T;
  double* vt = taps + ((ntaps + 1) & ~1);   // THX x TWX
  double* rt = vt + THX * TWX;              // THX x GT_W (horizontal pass)
  for (int t = threadIdx.x; t < ntaps; t += blockDim.x)
    taps[t] = sep ? (t < T ? a.av[t] : a.au[t - T]) : a.afull[t];
  const double* v = a.v.at(b, a.st);
  const int i0 = blockIdx.y * GT_H, j0 = blockIdx.x * GT_W;
  for (int idx = threadIdx.x; idx < THX * TWX; idx += blockDim.x) {
    const int ti = idx / TWX, tj = idx - ti * TWX;
    vt[idx] = v[(long long)wrap_fast(i0 - R + ti, H) * W + wrap_fast(j0 - R + tj, W)];
  }
  __syncthreads();
  if (sep) {
    for (int idx = threadIdx.x; idx < THX * GT_W; idx += blockDim.x) {
      const int ti = idx / GT_W, tj = idx - ti * GT_W;
      const double* row = vt + ti * TWX + tj;
      double s = 0.0;
      for (int d = 0; d < T; ++d) s = fma(taps[d], row[d], s);
      rt[idx] = s;
    }
    __syncthreads();
  }
  double* xo = a.gout ? nullptr : a.xout.at(b, a.st);
  const double* xp = a.gout ? nullptr : a.xprev.at(b, a.st);
  Acc acc;
  for (int idx = threadIdx.x; idx < GT_H * GT_W; idx += blockDim.x) {
    const int oi = idx / GT_W, oj = idx - oi * GT_W;
    const int gi = i0 + oi, gj = j0 + oj;
    if (gi >= H || gj >= W) continue;
    double hh = 0.0;
    if (sep) {
      const double* au = taps + T;
      for (int d = 0; d < T; ++d) hh = fma(au[d], rt[(oi + d) * GT_W + oj], hh);
    } else {
      for (int da = 0; da < T; ++da) {
        const double* row = vt + (oi + da) * TWX + oj;
        const double* tr = taps + da * T;
        for (int db = 0; db < T; ++db) hh = fma(tr[db], row[db], hh);
      }
    }
    const double vv = vt[(oi + R) * TWX + oj + R];
    grad_update(a, b, (long long)gi * W + gj, vv, hh, xo, xp, acc);
  }
  grad_finish(a, b, acc, gridDim.x * gridDim.y, blockIdx.y * gridDim.x + blockIdx.x);
}

// CG route: A v precomputed; hh = A v - alpha v so grad_update sees the same form.
__global__ void __launch_bounds__(GT_THREADS) k_grad_ew(GradArgs a) {
  const int b = blockIdx.y;
  if (!takes_step(a.st[b], a.ctl.phase)) return;
  const long long N = (long long)a.H * a.W;
  const double* v = a.v.at(b, a.st);
  double* xo = a.gout ? nullptr : a.xout.at(b, a.st);
  const double* xp = a.gout ? nullptr : a.xprev.at(b, a.st);
  const double* Av = a.Av + (long long)b * N;
  Acc acc;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    const double vv = v[i];
    grad_update(a, b, i, vv, fma(-a.alpha, vv, Av[i]), xo, xp, acc);
  }
  grad_finish(a, b, acc, gridDim.x, blockIdx.x);
}

static size_t stencil_smem(int R, bool sep) {
  const int T = 2 * R + 1, ntaps = sep ? 2 * T : T * T;
  return sizeof(double) * (((ntaps + 1) & ~1) + (size_t)(GT_H + 2 * R) * (GT_W + 2 * R) +
                           (sep ? (size_t)(GT_H + 2 * R) * GT_W : 0));
}

int grad_partials_per_image(int H, int W, bool stencil) {
  if (stencil) return cdivg(W, GT_W) * cdivg(H, GT_H);
  return ew_chunks((long long)H * W);
}

void launch_grad_step(const GradArgs& a, cudaStream_t s) {
  if (a.Av) {
    k_grad_ew<<<dim3(ew_chunks((long long)a.H * a.W), a.B), GT_THREADS, 0, s>>>(a);
    return;
  }
  const size_t sm = stencil_smem(a.R, a.au != nullptr);
  static size_t opted = 48 * 1024;
  if (sm > opted) {
    cudaFuncSetAttribute(k_grad_stencil, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    opted = sm;
  }
  k_grad_stencil<<<dim3(cdivg(a.W, GT_W), cdivg(a.H, GT_H), a.B), GT_THREADS, sm, s>>>(a);
}

}  // namespace redve
