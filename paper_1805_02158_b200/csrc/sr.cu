// Super-resolution path: PatchWeighted denoiser, fused BlurDownsample normal
// operator, scipy-exact conjugate gradients, generic step record (fp64).
//
// PatchWeighted (denoisers.py:49-129) with its balancing factorised: after
// t sweeps every map is w_o(p) = w0_o(p) D(p) D(p+o), D = prod of the sweep
// scalings, so a sweep only updates the scalar field
//     D(p) <- D(p) / sqrt( D(p) * sum_o w0_o(p) D(p+o) )
// and f(p) = D(p) sum_o w0_o(p) D(p+o) x(p+o).  Raw weights are symmetric,
// w0_{-o}(p) = w0_o(p-o), so only the 24 offsets of a half plane are stored.
//
// CG (scipy 1.18.1 sparse/linalg/_isolve/iterative.py:311-430 as called by
// objective.py:105-121): warm start x0 = x_k, stop when ||r|| < 1e-6 ||b||
// tested before every iteration, r updated recursively, maxiter 200, abort
// if the true residual exceeds 1e-4 ||rhs|| after maxiter.
#include "kernels.cuh"
#include "sr.cuh"

namespace redve {

extern __shared__ __align__(16) unsigned char s_smem[];

static inline int cdivs(long long a, long long b) { return (int)((a + b - 1) / b); }

// --------------------------------------------------------------- PatchWeighted
constexpr int PW_T = 32;  // output tile edge

__device__ __forceinline__ void pw_offset(int k, int sr, int& di, int& dj) {
  // k-th offset of the half plane {di > 0} U {di == 0, dj > 0}, raster order
  const int side = 2 * sr + 1;
  const int lin = (side * side + 1) / 2 + k;  // skip the centre and the negative half
  di = lin / side - sr;
  dj = lin % side - sr;
}

// w0_o(p) = exp(-max(box_{(2pr+1)^2} mean of (x(q)-x(q+o))^2, 0) / h^2)
__global__ void __launch_bounds__(256) k_pw_weights(PwArgs a) {
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W, pr = a.pr, sr = a.sr;
  const int halo = pr + sr;
  const int X = PW_T + 2 * halo;   // x tile edge
  const int E = PW_T + 2 * pr;     // squared-difference tile edge
  double* xs = reinterpret_cast<double*>(s_smem);
  double* es = xs + X * X;
  double* rs = es + E * E;
  const int i0 = blockIdx.y * PW_T, j0 = blockIdx.x * PW_T;
  const double* x = a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < X * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    xs[idx] = __ldg(x + (long long)wrap(i0 - halo + ti, H) * W + wrap(j0 - halo + tj, W));
  }
  __syncthreads();
  const long long N = (long long)H * W;
  const double inv_box = 1.0 / ((2 * pr + 1) * (2 * pr + 1));
  for (int k = 0; k < a.npos; ++k) {
    int di, dj;
    pw_offset(k, sr, di, dj);
    for (int idx = threadIdx.x; idx < E * E; idx += blockDim.x) {
      const int ei = idx / E, ej = idx - ei * E;
      const int ti = ei + sr, tj = ej + sr;  // tile coords of q
      const double d = xs[ti * X + tj] - xs[(ti + di) * X + tj + dj];
      es[idx] = d * d;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < E * PW_T; idx += blockDim.x) {
      const int ei = idx / PW_T, oj = idx - ei * PW_T;
      double s = 0.0;
      for (int t = 0; t < 2 * pr + 1; ++t) s += es[ei * E + oj + t];
      rs[idx] = s;
    }
    __syncthreads();
    double* w0 = a.w0 + ((long long)b * a.npos + k) * N;
    for (int idx = threadIdx.x; idx < PW_T * PW_T; idx += blockDim.x) {
      const int oi = idx / PW_T, oj = idx - oi * PW_T;
      const int gi = i0 + oi, gj = j0 + oj;
      if (gi >= H || gj >= W) continue;
      double s = 0.0;
      for (int t = 0; t < 2 * pr + 1; ++t) s += rs[(oi + t) * PW_T + oj];
      const double d2 = s * inv_box;
      w0[(long long)gi * W + gj] = exp(-fmax(d2, 0.0) * a.inv_h2);
    }
    __syncthreads();
  }
}

// One balancing sweep (apply = 0) or the final application (apply = 1):
//   S(p) = v(p) + sum_{o in half plane} [ w0_o(p) v(p+o) + w0_o(p-o) v(p-o) ]
// with v = D (sweep) or v = D x (apply); D_new = D / sqrt(D S), f = D S.
__global__ void __launch_bounds__(256) k_pw_sweep(PwArgs a, const double* Din, double* Dout,
                                                  int first, int apply) {
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W, sr = a.sr;
  const int X = PW_T + 2 * sr;
  double* vs = reinterpret_cast<double*>(s_smem);
  const int i0 = blockIdx.y * PW_T, j0 = blockIdx.x * PW_T;
  const long long N = (long long)H * W;
  const double* Db = Din + (long long)b * N;
  const double* x = apply ? a.xin.at(b, a.st) : nullptr;
  for (int idx = threadIdx.x; idx < X * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    const long long o = (long long)wrap(i0 - sr + ti, H) * W + wrap(j0 - sr + tj, W);
    const double d = first ? 1.0 : __ldg(Db + o);
    vs[idx] = apply ? d * __ldg(x + o) : d;
  }
  __syncthreads();
  const double* w0b = a.w0 + (long long)b * a.npos * N;
  for (int idx = threadIdx.x; idx < PW_T * PW_T; idx += blockDim.x) {
    const int oi = idx / PW_T, oj = idx - oi * PW_T;
    const int gi = i0 + oi, gj = j0 + oj;
    if (gi >= H || gj >= W) continue;
    const int ci = oi + sr, cj = oj + sr;
    double S = vs[ci * X + cj];
    for (int k = 0; k < a.npos; ++k) {
      int di, dj;
      pw_offset(k, sr, di, dj);
      const double* w0 = w0b + (long long)k * N;
      const double wp = __ldg(w0 + (long long)gi * W + gj);
      const double wm = __ldg(w0 + (long long)wrap(gi - di, H) * W + wrap(gj - dj, W));
      S = fma(wp, vs[(ci + di) * X + cj + dj], S);
      S = fma(wm, vs[(ci - di) * X + cj - dj], S);
    }
    const long long o = (long long)gi * W + gj;
    const double d = first ? 1.0 : Db[o];
    if (apply) {
      a.out[(long long)b * N + o] = d * S;
    } else {
      Dout[(long long)b * N + o] = d / sqrt(d * S);
    }
  }
}

// Balanced maps of every offset, raster order (denoisers.py:83-111):
// maps[k](p) = w0_o(p) D(p) D(p+o), w0_{-o}(p) = w0_o(p-o), w0_0 = 1.
__global__ void k_pw_maps(PwArgs a, const double* D, double* maps) {
  const int b = blockIdx.y;
  const int H = a.H, W = a.W, sr = a.sr, side = 2 * sr + 1;
  const long long N = (long long)H * W;
  const double* Db = D + (long long)b * N;
  const double* w0b = a.w32 ? reinterpret_cast<const double*>(
                                  reinterpret_cast<const float*>(a.w0) + (long long)b * a.npos * N)
                            : a.w0 + (long long)b * a.npos * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / W), j = (int)(idx - (long long)i * W);
    for (int lin = 0; lin < side * side; ++lin) {
      const int di = lin / side - sr, dj = lin % side - sr;
      const int center = (side * side - 1) / 2;
      double w;
      long long wi = -1;
      if (lin > center) {
        wi = (long long)(lin - center - 1) * N + idx;
      } else if (lin < center) {  // negative offset: mirror plane, evaluated at p + o
        const int k = (side * side - 1 - lin) - center - 1;
        wi = (long long)k * N + (long long)wrap(i + di, H) * W + wrap(j + dj, W);
      }
      if (wi < 0) w = 1.0;
      else w = a.w32 ? (double)reinterpret_cast<const float*>(w0b)[wi] : w0b[wi];
      const double dq = Db[(long long)wrap(i + di, H) * W + wrap(j + dj, W)];
      maps[((long long)b * side * side + lin) * N + idx] = w * Db[idx] * dq;
    }
  }
}

// ---- compile-time specialisations (the generic kernels above serve any radii).
// Offsets are constants after unrolling, tiles have compile-time edges, and
// blocks whose halo stays inside the image skip the periodic index wrap.

template <int SR>
struct HalfPlane {
  static constexpr int SIDE = 2 * SR + 1;
  static constexpr int NPOS = (SIDE * SIDE - 1) / 2;
  __host__ __device__ static constexpr int di(int k) { return ((SIDE * SIDE + 1) / 2 + k) / SIDE - SR; }
  __host__ __device__ static constexpr int dj(int k) { return ((SIDE * SIDE + 1) / 2 + k) % SIDE - SR; }
};

constexpr int PW_ROWS = 4;  // output rows per thread (a column strip), 256 threads = 32 x 8 strips

// Raw weights: every thread owns a 4-row column strip of the 32x32 tile and
// keeps the (4+2PR) x (2PR+1) patch of x around it in registers; for each
// offset it forms the squared differences, the separable box sums and the
// exponential without any block synchronisation.
// exp of the (fp64) weight argument in the plane's precision: fp32 planes
// take the single-precision exp (within 2 fp32 ulp of the rounded fp64 value)
template <typename WT>
__device__ __forceinline__ WT pw_weight(double arg);
template <>
__device__ __forceinline__ double pw_weight<double>(double arg) { return exp(arg); }
template <>
__device__ __forceinline__ float pw_weight<float>(double arg) { return expf((float)arg); }

template <int PR, int SR, typename WT>
__global__ void __launch_bounds__(256) k_pw_weights_t(PwArgs a) {
  constexpr int HALO = PR + SR, X = PW_T + 2 * HALO, P = 2 * PR + 1, R = PW_ROWS + 2 * PR;
  constexpr int NP = HalfPlane<SR>::NPOS;
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W;
  double* xs = reinterpret_cast<double*>(s_smem);
  const int i0 = blockIdx.y * PW_T, j0 = blockIdx.x * PW_T;
  const double* x = a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < X * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    xs[idx] = __ldg(x + (long long)wrap_fast(i0 - HALO + ti, H) * W + wrap_fast(j0 - HALO + tj, W));
  }
  __syncthreads();
  const int oj = threadIdx.x & (PW_T - 1);
  const int oi0 = (threadIdx.x >> 5) * PW_ROWS;
  const int gj = j0 + oj;
  if (gj >= W || i0 + oi0 >= H) return;
  // tile coordinates of the strip's top-left patch element q = p + (-PR, -PR)
  const int ti0 = oi0 + HALO - PR, tj0 = oj + HALO - PR;
  double xc[R][P];
#pragma unroll
  for (int u = 0; u < R; ++u)
#pragma unroll
    for (int v = 0; v < P; ++v) xc[u][v] = xs[(ti0 + u) * X + tj0 + v];
  const long long N = (long long)H * W;
  const double inv_box = 1.0 / (P * P);
  WT* w0 = reinterpret_cast<WT*>(a.w0) + (long long)b * NP * N + (long long)(i0 + oi0) * W + gj;
  const int rows = min(PW_ROWS, H - (i0 + oi0));
#pragma unroll 2
  for (int k = 0; k < NP; ++k) {
    const int di = HalfPlane<SR>::di(k), dj = HalfPlane<SR>::dj(k);
    double rs[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      double acc = 0.0;
#pragma unroll
      for (int v = 0; v < P; ++v) {
        const double d = xc[u][v] - xs[(ti0 + u + di) * X + tj0 + v + dj];
        acc += d * d;
      }
      rs[u] = acc;
    }
#pragma unroll
    for (int m = 0; m < PW_ROWS; ++m) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < P; ++t) s += rs[m + t];
      if (m < rows) w0[(long long)k * N + (long long)m * W] = pw_weight<WT>(-fmax(s * inv_box, 0.0) * a.inv_h2);
    }
  }
}

// Balancing sweep / application with compile-time offsets:
//   S(p) = v(p) + sum_k [ w0_k(p) v(p+o_k) + w0_k(p-o_k) v(p-o_k) ]
template <int SR, int RPT, typename WT>
__global__ void __launch_bounds__(256, RPT == 1 ? 6 : 1)  // 40 registers: 538 vs 558 us per 768^2 call at 4 CTAs/SM
    k_pw_sweep_t(PwArgs a, const double* Din, double* Dout,
                                                    int first, int apply) {
  // tile: 32 columns x TH = 8*RPT rows (RPT rows per thread; fewer for small
  // images so the grid still fills the GPU)
  constexpr int X = PW_T + 2 * SR, TH = 8 * RPT, Y = TH + 2 * SR, NP = HalfPlane<SR>::NPOS;
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W;
  double* vs = reinterpret_cast<double*>(s_smem);
  const int i0 = blockIdx.y * TH, j0 = blockIdx.x * PW_T;
  const long long N = (long long)H * W;
  const double* Db = Din + (long long)b * N;
  const double* x = apply ? a.xin.at(b, a.st) : nullptr;
  for (int idx = threadIdx.x; idx < Y * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    const long long o = (long long)wrap_fast(i0 - SR + ti, H) * W + wrap_fast(j0 - SR + tj, W);
    const double d = first ? 1.0 : __ldg(Db + o);
    vs[idx] = apply ? d * __ldg(x + o) : d;
  }
  __syncthreads();
  const bool interior = i0 >= SR && j0 >= SR && i0 + TH + SR <= H && j0 + PW_T + SR <= W;
  const WT* w0b = reinterpret_cast<const WT*>(a.w0) + (long long)b * NP * N;
  const int oj = threadIdx.x & (PW_T - 1);
  const int gj = j0 + oj;
  if (gj >= W) return;
  // the block's 8 warps cover 8 consecutive rows per step m, so the rows above
  // that the mirrored loads w0_k(p - o_k) touch were fetched a step earlier;
  // the 4 rows of a thread are accumulated together for memory-level parallelism
  const int cj = oj + SR;
  int gi[RPT], ci[RPT];
  long long o[RPT];
  double S[RPT];
#pragma unroll
  for (int m = 0; m < RPT; ++m) {
    const int oi = (threadIdx.x >> 5) + 8 * m;
    gi[m] = min(i0 + oi, H - 1);  // rows past the image edge compute a throwaway copy
    ci[m] = gi[m] - i0 + SR;
    o[m] = (long long)gi[m] * W + gj;
    S[m] = vs[ci[m] * X + cj];
  }
  if (interior) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int di = HalfPlane<SR>::di(k), dj = HalfPlane<SR>::dj(k);
      const WT* wk = w0b + (long long)k * N;
      const int sh = di * W + dj;
      double wp[RPT], wm[RPT];
#pragma unroll
      for (int m = 0; m < RPT; ++m) {
        wp[m] = (double)__ldg(wk + o[m]);
        wm[m] = (double)__ldg(wk + o[m] - sh);
      }
#pragma unroll
      for (int m = 0; m < RPT; ++m) {
        S[m] = fma(wp[m], vs[(ci[m] + di) * X + cj + dj], S[m]);
        S[m] = fma(wm[m], vs[(ci[m] - di) * X + cj - dj], S[m]);
      }
    }
  } else {
#pragma unroll 1
    for (int k = 0; k < NP; ++k) {
      const int di = HalfPlane<SR>::di(k), dj = HalfPlane<SR>::dj(k);
      const WT* wk = w0b + (long long)k * N;
      const int cm = wrap_fast(gj - dj, W);
#pragma unroll
      for (int m = 0; m < RPT; ++m) {
        const double wp = (double)__ldg(wk + o[m]);
        const double wm = (double)__ldg(wk + (long long)wrap_fast(gi[m] - di, H) * W + cm);
        S[m] = fma(wp, vs[(ci[m] + di) * X + cj + dj], S[m]);
        S[m] = fma(wm, vs[(ci[m] - di) * X + cj - dj], S[m]);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < RPT; ++m) {
    if (i0 + (int)(threadIdx.x >> 5) + 8 * m >= H) break;
    const double d = first ? 1.0 : Db[o[m]];
    if (apply) a.out[(long long)b * N + o[m]] = d * S[m];
    else Dout[(long long)b * N + o[m]] = d / sqrt(d * S[m]);
  }
}

// Vectorised sweep: each thread owns VW = 16 / sizeof(WT) adjacent outputs of
// one row, so every plane read is a 16-byte load (4 fp32 or 2 fp64 weights).
// The sweep is bound by outstanding load requests, not bytes (ncu: long-
// scoreboard stalls at 3.1 TB/s for both plane widths with one output per
// thread), so fewer, wider requests are what moves it toward the HBM roof.
// The mirrored weight w0_k(p - o_k) starts -dj columns off the vector grid:
// for dj % VW != 0 it is spliced from two aligned loads (compile-time lanes).
template <int VW>
struct VecSplit {  // q = -dj split as VW * qb + qr, 0 <= qr < VW
  __host__ __device__ static constexpr int qb(int q) { return q >= 0 ? q / VW : -((-q + VW - 1) / VW); }
  __host__ __device__ static constexpr int qr(int q) { return q - VW * qb(q); }
};

template <typename WT>
union WVec {
  int4 raw;
  WT e[16 / sizeof(WT)];
};

// Shared D tile of the vector sweep: the columns of a row are stored as VW
// interleaved sub-rows (column c at (c % VW) * SUB + c / VW), so the 32 lanes
// of a warp, whose columns are VW apart, read consecutive doubles (the plain
// row layout is a 4-way bank conflict on every one of the 2 NP VW reads).
// 1 / sqrt(a), a > 0 finite: MUFU.RSQ64H seed (~20 bits) + two Newton steps
// (relative error ~1e-24 before the final rounding) -- 12 instructions where
// sqrt + division take ~60; the balancing update then is d * rsqrt(d S),
// within 2 ulp of d / sqrt(d S).
__device__ __forceinline__ double pw_rsqrt(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

template <int SR, int VW>
struct VTile {
  static constexpr int X = 32 * VW + 2 * SR, SUB = (X + VW - 1) / VW, XS = VW * SUB;
  __device__ static __forceinline__ int at(int row, int col) { return row * XS + (col % VW) * SUB + col / VW; }
};

// What each stage costs was measured on a stand-alone rebuild of this kernel
// (tools/pw_sweep_probe.cu, DESIGN 3.4): the plane loads, converts and FMAs
// alone run at the HBM roof; the tile prologue, the shared reads and the
// epilogue each add time that does not overlap.  Hence: the tile arrives by
// cp.async (one round trip instead of load -> store pairs), the first offset's
// plane vectors are requested before the prologue's wait, the tile is bank-
// conflict free, the epilogue takes d from the tile, 4 CTAs/SM (64 registers).
template <int SR, typename WT, int TH = 8>  // TH tile rows = warps per CTA
__global__ void __launch_bounds__(32 * TH, 32 / TH)  // 1024 threads/SM (64 registers)
    k_pw_sweep_v(PwArgs a, const double* Din, double* Dout,
                                                    int first, int apply) {
  constexpr int VW = 16 / sizeof(WT), TW = 32 * VW;
  constexpr int X = TW + 2 * SR, Y = TH + 2 * SR, NP = HalfPlane<SR>::NPOS;
  using VT = VTile<SR, VW>;
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W;
  double* vs = reinterpret_cast<double*>(s_smem);
  const int i0 = blockIdx.y * TH, j0 = blockIdx.x * TW;
  const long long N = (long long)H * W;
  const double* Db = Din + (long long)b * N;
  const double* x = apply ? a.xin.at(b, a.st) : nullptr;
  const int lane = threadIdx.x & 31, oi = threadIdx.x >> 5;
  const int gj = j0 + VW * lane;
  const int gi = min(i0 + oi, H - 1);  // rows past the image edge compute a throwaway copy
  const int ci = gi - i0 + SR;
  const long long o = (long long)gi * W + gj;
  const WT* w0b = reinterpret_cast<const WT*>(a.w0) + (long long)b * NP * N;
  const bool interior = i0 >= SR && i0 + TH + SR <= H && j0 >= 2 * VW && j0 + TW + 2 * VW <= W;
  WVec<WT> wp0, lo0, hi0;  // offset 0 = (0, 1): requested before the tile is waited for
  if (interior) {
    constexpr int dj0 = HalfPlane<SR>::dj(0);
    static_assert(HalfPlane<SR>::di(0) == 0 && VecSplit<VW>::qr(-dj0) != 0, "first offset is (0, 1)");
    wp0.raw = __ldg(reinterpret_cast<const int4*>(w0b + o));
    const long long om = o + VW * VecSplit<VW>::qb(-dj0);
    lo0.raw = __ldg(reinterpret_cast<const int4*>(w0b + om));
    hi0.raw = __ldg(reinterpret_cast<const int4*>(w0b + om + VW));
  }
  for (int idx = threadIdx.x; idx < Y * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    const long long q = (long long)wrap_fast(i0 - SR + ti, H) * W + wrap_fast(j0 - SR + tj, W);
    double* dst = vs + VT::at(ti, tj);
    if (first) {
      *dst = apply ? __ldg(x + q) : 1.0;
    } else if (apply) {
      *dst = __ldg(Db + q) * __ldg(x + q);
    } else {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
                   "l"(Db + q));
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (gj >= W) return;
  // v(row, m): tile row `row`, column VW * lane + m (m a compile-time constant)
#define PW_V(row, m) vs[(row)*VT::XS + ((m) % VW) * VT::SUB + (m) / VW + lane]
  double S[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) S[t] = PW_V(ci, SR + t);
  if (interior) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int di = HalfPlane<SR>::di(k), dj = HalfPlane<SR>::dj(k);
      const WT* wk = w0b + (long long)k * N;
      WVec<WT> wp, lo, hi;
      if (k == 0) {
        wp = wp0;
        lo = lo0;
        hi = hi0;
      } else {
        wp.raw = __ldg(reinterpret_cast<const int4*>(wk + o));
        const long long om = o - (long long)di * W + VW * VecSplit<VW>::qb(-dj);
        lo.raw = __ldg(reinterpret_cast<const int4*>(wk + om));
        if (VecSplit<VW>::qr(-dj) != 0) hi.raw = __ldg(reinterpret_cast<const int4*>(wk + om + VW));
        else hi.raw = lo.raw;
      }
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        const int u = t + VecSplit<VW>::qr(-dj);
        const double wm = (double)(u < VW ? lo.e[u < VW ? u : 0] : hi.e[u >= VW ? u - VW : 0]);
        S[t] = fma((double)wp.e[t], PW_V(ci + di, SR + t + dj), S[t]);
        S[t] = fma(wm, PW_V(ci - di, SR + t - dj), S[t]);
      }
    }
  } else {
    // tiles on the periodic seam: the same vector loads with wrapped rows and
    // vector columns (W % VW == 0: an aligned vector never straddles the seam)
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int di = HalfPlane<SR>::di(k), dj = HalfPlane<SR>::dj(k);
      const WT* wk = w0b + (long long)k * N;
      const long long rm = (long long)wrap_fast(gi - di, H) * W;
      const int cl = gj + VW * VecSplit<VW>::qb(-dj);
      WVec<WT> wp, lo, hi;
      wp.raw = __ldg(reinterpret_cast<const int4*>(wk + o));
      lo.raw = __ldg(reinterpret_cast<const int4*>(wk + rm + wrap_fast(cl, W)));
      if (VecSplit<VW>::qr(-dj) != 0) hi.raw = __ldg(reinterpret_cast<const int4*>(wk + rm + wrap_fast(cl + VW, W)));
      else hi.raw = lo.raw;
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        const int u = t + VecSplit<VW>::qr(-dj);
        const double wm = (double)(u < VW ? lo.e[u < VW ? u : 0] : hi.e[u >= VW ? u - VW : 0]);
        S[t] = fma((double)wp.e[t], PW_V(ci + di, SR + t + dj), S[t]);
        S[t] = fma(wm, PW_V(ci - di, SR + t - dj), S[t]);
      }
    }
  }
  if (i0 + oi >= H) return;
#pragma unroll
  for (int t = 0; t < VW; ++t) {
    // the tile holds D itself on a balancing sweep (the same value as Db[o + t])
    const double d = first ? 1.0 : (apply ? Db[o + t] : PW_V(ci, SR + t));
    if (apply) a.out[(long long)b * N + o + t] = d * S[t];
    else Dout[(long long)b * N + o + t] = d * pw_rsqrt(d * S[t]);
  }
#undef PW_V
}

template <int SR, typename WT, int TH>
static void pw_sweeps_v(const PwArgs& a, cudaStream_t s, int* launches, bool with_apply) {
  constexpr int VW = 16 / sizeof(WT), TW = 32 * VW;
  dim3 grid(cdivs(a.W, TW), cdivs(a.H, TH), a.B);
  const size_t sm = sizeof(double) * VTile<SR, VW>::XS * (TH + 2 * SR);
  const double* din = a.D0;
  double* dout = a.D1;
  for (int it = 0; it < a.iters; ++it) {
    k_pw_sweep_v<SR, WT, TH><<<grid, 32 * TH, sm, s>>>(a, din, dout, it == 0, 0);
    ++*launches;
    din = dout;
    dout = (dout == a.D1) ? a.D0 : a.D1;
  }
  if (with_apply) {
    k_pw_sweep_v<SR, WT, TH><<<grid, 32 * TH, sm, s>>>(a, din, nullptr, a.iters == 0, 1);
    ++*launches;
  }
}

template <int SR, int RPT, typename WT>
static void pw_sweeps_t(const PwArgs& a, cudaStream_t s, int* launches, bool with_apply) {
  dim3 grid(cdivs(a.W, PW_T), cdivs(a.H, 8 * RPT), a.B);
  const size_t sm = sizeof(double) * (PW_T + 2 * SR) * (8 * RPT + 2 * SR);
  const double* din = a.D0;
  double* dout = a.D1;
  for (int it = 0; it < a.iters; ++it) {
    k_pw_sweep_t<SR, RPT, WT><<<grid, 256, sm, s>>>(a, din, dout, it == 0, 0);
    ++*launches;
    din = dout;
    dout = (dout == a.D1) ? a.D0 : a.D1;
  }
  if (with_apply) {
    k_pw_sweep_t<SR, RPT, WT><<<grid, 256, sm, s>>>(a, din, nullptr, a.iters == 0, 1);
    ++*launches;
  }
}

template <int PR, int SR, typename WT>
static void pw_pass_t(const PwArgs& a, cudaStream_t s, int* launches, bool with_apply) {
  dim3 grid(cdivs(a.W, PW_T), cdivs(a.H, PW_T), a.B);
  constexpr int X = PW_T + 2 * (PR + SR);
  k_pw_weights_t<PR, SR, WT><<<grid, 256, sizeof(double) * X * X, s>>>(a);
  ++*launches;
  // rows per thread: 1 measured best at every size (768^2: 0.91 ms vs 1.30 ms
  // with 4; 4096^2: 14.7 vs 21.8 ms) -- more, smaller CTAs hide the latency
  int rpt = 1;
  if (const char* e = getenv("REDVE_PW_RPT")) rpt = atoi(e);  // experiments
  // the vector sweep (16-byte plane loads, cp.async tile, conflict-free tile
  // layout, vector loads on the seam tiles too) is the faster one wherever it
  // applies: per call 768^2 fp32 0.64 -> 0.47 ms, 512^2 0.42 -> 0.37, 2048^2
  // 3.19 -> 2.74, fp64 planes 0.88 -> 0.76 at 768^2; level below 384^2 where
  // the 22 launches dominate (tools/gpu_pw_sizes.sh)
  constexpr int VW = 16 / (int)sizeof(WT);
  bool vec = a.W % VW == 0 && a.W >= 32 * VW;
  if (const char* e = getenv("REDVE_PW_VEC")) vec = e[0] == '1' ? (a.W % VW == 0 && a.W >= 32 * VW)
                                                                : false;
  if (vec) {
    // 16-row tiles (512 threads): 1.375x instead of 1.75x of the D tile is halo and
    // fewer mirrored rows fall outside the CTA: 365 -> 360 us per 768^2 call,
    // 38.1 -> 37.6 ms per 8192^2 call
    int th = a.H >= 64 ? 16 : 8;
    if (const char* e = getenv("REDVE_PW_TH")) th = atoi(e);  // experiments
    if (th == 16) pw_sweeps_v<SR, WT, 16>(a, s, launches, with_apply);
    else pw_sweeps_v<SR, WT, 8>(a, s, launches, with_apply);
    return;
  }
  if (rpt == 4) pw_sweeps_t<SR, 4, WT>(a, s, launches, with_apply);
  else if (rpt == 2) pw_sweeps_t<SR, 2, WT>(a, s, launches, with_apply);
  else pw_sweeps_t<SR, 1, WT>(a, s, launches, with_apply);
}

// true if a specialisation ran; the final D is in D0 if iters is even, else D1
static bool pw_specialised(const PwArgs& a, cudaStream_t s, int* launches, bool with_apply) {
#define PW_CASE(PRV, SRV)                                  \
  if (a.pr == PRV && a.sr == SRV) {                        \
    if (a.w32) pw_pass_t<PRV, SRV, float>(a, s, launches, with_apply);  \
    else pw_pass_t<PRV, SRV, double>(a, s, launches, with_apply);      \
    return true;                                           \
  }
  PW_CASE(1, 3) PW_CASE(1, 1) PW_CASE(1, 2) PW_CASE(0, 3) PW_CASE(2, 3) PW_CASE(0, 1)
#undef PW_CASE
  return false;
}

void launch_pw_maps(const PwArgs& a_in, cudaStream_t s, int* launches, double* maps) {
  dim3 grid(cdivs(a_in.W, PW_T), cdivs(a_in.H, PW_T), a_in.B);
  PwArgs a = a_in;
  const double* din = a.D0;
  if (pw_specialised(a, s, launches, false)) {
    din = (a.iters % 2 == 0) ? a.D0 : a.D1;
  } else {
    a.w32 = 0;  // the generic kernels keep fp64 planes
    k_pw_weights<<<grid, 256, pw_weights_smem(a.pr, a.sr), s>>>(a);
    const size_t sm = sizeof(double) * (PW_T + 2 * a.sr) * (PW_T + 2 * a.sr);
    double* dout = a.D1;
    for (int it = 0; it < a.iters; ++it) {
      k_pw_sweep<<<grid, 256, sm, s>>>(a, din, dout, it == 0, 0);
      din = dout;
      dout = (dout == a.D1) ? a.D0 : a.D1;
    }
    *launches += a.iters + 1;
  }
  k_pw_maps<<<dim3(cdivs((long long)a.H * a.W, 256), a.B), 256, 0, s>>>(a, din, maps);
  ++*launches;
}

size_t pw_weights_smem(int pr, int sr) {
  const int X = PW_T + 2 * (pr + sr), E = PW_T + 2 * pr;
  return sizeof(double) * ((size_t)X * X + (size_t)E * E + (size_t)E * PW_T);
}

void launch_pw(const PwArgs& a_in, cudaStream_t s, int* launches) {
  if (pw_specialised(a_in, s, launches, true)) return;
  PwArgs a = a_in;
  a.w32 = 0;  // the generic kernels keep fp64 planes
  dim3 grid(cdivs(a.W, PW_T), cdivs(a.H, PW_T), a.B);
  k_pw_weights<<<grid, 256, pw_weights_smem(a.pr, a.sr), s>>>(a);
  ++*launches;
  const size_t sm = sizeof(double) * (PW_T + 2 * a.sr) * (PW_T + 2 * a.sr);
  const double* din = a.D0;
  double* dout = a.D1;
  for (int it = 0; it < a.iters; ++it) {
    k_pw_sweep<<<grid, 256, sm, s>>>(a, din, dout, it == 0, 0);
    ++*launches;
    din = dout;
    dout = (dout == a.D1) ? a.D0 : a.D1;
  }
  k_pw_sweep<<<grid, 256, sm, s>>>(a, din, nullptr, a.iters == 0, 1);
  ++*launches;
}

// --------------------------------------------------------------- normal operator
// (A w)(u,v) = (1/sigma^2) (H^T H w)(u,v) + alpha w(u,v),  H = keep(== 0 mod s) o conv.
// Tile: TH x TW outputs, w tile with halo 2r in shared memory.  Only the
// measurement-lattice samples of z = H w inside the tile's reach are formed
// (a compact lattice list, periodic seams included), and each output gathers
// the <= ceil((2r+1)/s)^2 lattice samples in its window -- the same terms, in
// the same order, as the dense correlation with the zero-filled z_up.
// the matvec passes' reduced sums -> CG state (scipy cg, iterative.py:384-430)
template <int MODE>
__device__ __forceinline__ void cg_reduce_finish(CgState& cs, const CgArgs& a, int b, double t0,
                                                 double t1) {
  if (MODE == CG_ITER) {
    cs.alpha = cs.rho / t0;  // rho_cur / (p . q)
  } else if (MODE == CG_INIT) {
    const double bn = sqrt(t0);
    cs.bn2 = t0;
    cs.atol = a.rtol * bn;  // max(atol=0, rtol*||b||)
    cs.rho = t1;
    cs.its = 0;
    cs.info = 0;
    cs.need_resid = 0;
    cs.zero_b = (bn == 0.0);
    cs.active = !(cs.zero_b || sqrt(t1) < cs.atol);
  } else {  // residual check after maxiter (objective.py:114-120)
    if (sqrt(t1) > a.abort * sqrt(t0)) a.st[b].err = ERR_CG;
    cs.need_resid = 0;
  }
}

constexpr int MV_TH = 32, MV_TW = 32;

template <int MODE>
__global__ void __launch_bounds__(256) k_cg_matvec(CgArgs a) {
  const int b = blockIdx.z;
  CgState& cs = a.cg[b];
  if (MODE == CG_INIT) {
    if (!takes_step(a.st[b], a.phase)) return;
  } else if (MODE == CG_ITER) {
    if (!cs.active) return;
  } else if (MODE == CG_RESID) {
    if (!takes_step(a.st[b], a.phase) || !cs.need_resid) return;
  }
  const int H = a.H, W = a.W, s = a.factor, k = a.k, r = k / 2;
  const int WX = MV_TW + 4 * r, HX = MV_TH + 4 * r;  // w tile
  const int WZ = MV_TW + 2 * r, HZ = MV_TH + 2 * r;  // z_up window
  double* taps = reinterpret_cast<double*>(s_smem);
  double* ws = taps + k * k;
  double* zc = ws + HX * WX;                // compact lattice samples [nzr][nzc]
  double* red = zc + HZ * WZ;
  int* zr_pos = reinterpret_cast<int*>(red + 64);  // lattice rows / cols (window coords)
  int* zc_pos = zr_pos + HZ;
  int* rwin = zc_pos + WZ;                  // per output row: first lattice row, count
  int* cwin = rwin + 2 * MV_TH;             // (rwin doubles as flag scratch: >= 64 + WZ ints)
  __shared__ int s_nzr, s_nzc;
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) taps[i] = a.taps[i];
  const long long N = (long long)H * W;
  const int i0 = blockIdx.y * MV_TH, j0 = blockIdx.x * MV_TW;
  const bool cont = MODE == CG_ITER && cs.its > 0;  // p = r + beta p_old after the 1st iteration
  const double beta = cont ? cs.beta : 0.0;
  const double* rr = a.r + (long long)b * N;
  const double* pold = a.p + (long long)b * N;
  const double* xin = (MODE == CG_ITER) ? nullptr : a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < HX * WX; idx += blockDim.x) {
    const int ti = idx / WX, tj = idx - ti * WX;
    const long long o =
        (long long)wrap_fast(i0 - 2 * r + ti, H) * W + wrap_fast(j0 - 2 * r + tj, W);
    double w;
    if (MODE == CG_ITER) w = cont ? fma(beta, pold[o], rr[o]) : rr[o];
    else w = xin[o];
    ws[idx] = w;
  }
  // lattice rows / columns of the window: measurement lattice by GLOBAL row
  // (a slab of a spatially split image starts at global row a.row0 of an
  // a.Hg-row image)
  int* flag = rwin;  // scratch: lattice flags of window rows [0, HZ) and columns [64, 64 + WZ)
  if (threadIdx.x < HZ) {
    const int gu = wrap_fast(i0 - r + (int)threadIdx.x, H);
    const int gg = (a.Hg > 0) ? (int)(((long long)a.row0 + gu) % a.Hg) : gu;
    flag[threadIdx.x] = (gg % s) == 0;
  } else if (threadIdx.x >= 64 && threadIdx.x < 64 + WZ) {
    flag[threadIdx.x] = (wrap_fast(j0 - r + (int)threadIdx.x - 64, W) % s) == 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int zi = 0; zi < HZ; ++zi)
      if (flag[zi]) zr_pos[n++] = zi;
    s_nzr = n;
  } else if (threadIdx.x == 32) {
    int n = 0;
    for (int zj = 0; zj < WZ; ++zj)
      if (flag[64 + zj]) zc_pos[n++] = zj;
    s_nzc = n;
  }
  __syncthreads();
  const int nzr = s_nzr, nzc = s_nzc;
  // output row u (tile coords) reads window rows [u, u + 2r]
  if (threadIdx.x < MV_TH) {
    const int u = threadIdx.x;
    int first = 0;
    while (first < nzr && zr_pos[first] < u) ++first;
    int last = first;
    while (last < nzr && zr_pos[last] <= u + 2 * r) ++last;
    rwin[2 * u] = first;
    rwin[2 * u + 1] = last - first;
  } else if (threadIdx.x >= 64 && threadIdx.x < 64 + MV_TW) {
    const int v = threadIdx.x - 64;
    int first = 0;
    while (first < nzc && zc_pos[first] < v) ++first;
    int last = first;
    while (last < nzc && zc_pos[last] <= v + 2 * r) ++last;
    cwin[2 * v] = first;
    cwin[2 * v + 1] = last - first;
  }
  // z = H w at the lattice samples
  for (int idx = threadIdx.x; idx < nzr * nzc; idx += blockDim.x) {
    const int li = idx / nzc, lj = idx - li * nzc;
    const int zi = zr_pos[li], zj = zc_pos[lj];
    double z = 0.0;
    for (int ta = 0; ta < k; ++ta)
      for (int tb = 0; tb < k; ++tb)
        z = fma(taps[ta * k + tb], ws[(zi + r - (ta - r)) * WX + (zj + r - (tb - r))], z);
    zc[idx] = z;
  }
  __syncthreads();
  double acc[2] = {0.0, 0.0};
  const double inv_s2 = a.inv_sigma2;
  for (int idx = threadIdx.x; idx < MV_TH * MV_TW; idx += blockDim.x) {
    const int oi = idx / MV_TW, oj = idx - oi * MV_TW;
    const int gi = i0 + oi, gj = j0 + oj;
    if (gi >= H || gj >= W) continue;
    double ht = 0.0;  // (H^T z_up)(u, v): correlation over the window's lattice samples
    const int rf = rwin[2 * oi], rn = rwin[2 * oi + 1];
    const int cf = cwin[2 * oj], cn = cwin[2 * oj + 1];
    for (int i = rf; i < rf + rn; ++i) {
      const double* trow = taps + (zr_pos[i] - oi) * k - oj;
      const double* zrow = zc + i * nzc;
      for (int j = cf; j < cf + cn; ++j) ht = fma(trow[zc_pos[j]], zrow[j], ht);
    }
    const double wv = ws[(oi + 2 * r) * WX + (oj + 2 * r)];
    const double aw = fma(ht, inv_s2, a.alpha * wv);
    const long long o = (long long)b * N + (long long)gi * W + gj;
    if (MODE == CG_PLAIN) {
      a.q[o] = aw;
      continue;
    }
    if (MODE == CG_ITER) {
      a.p[o] = wv;
      a.q[o] = aw;
      acc[0] = fma(wv, aw, acc[0]);
    } else {
      const double bb = fma(a.alpha, a.f[o], a.hty[o]);  // rhs = H^T y/sigma^2 + alpha f
      const double res = bb - aw;
      if (MODE == CG_INIT) {
        a.r[o] = res;
        a.xout.at(b, a.st)[(long long)gi * W + gj] = wv;  // warm start copy x <- x_k
      }
      acc[0] = fma(bb, bb, acc[0]);
      acc[1] = fma(res, res, acc[1]);
    }
  }
  if (MODE == CG_PLAIN) return;
  block_sum<2>(acc, red);
  const int nblk = gridDim.x * gridDim.y;
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    a.partials[((long long)b * nblk + blk) * 2] = acc[0];
    a.partials[((long long)b * nblk + blk) * 2 + 1] = acc[1];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double tt[2];
  if (lastb) gather_partials<2>(a.partials + (long long)b * nblk * 2, nblk, tt, red);
  if (lastb && threadIdx.x == 0) cg_reduce_finish<MODE>(cs, a, b, tt[0], tt[1]);
}

// Compile-time operator (7 x 7 PSF, factor 3: configs[2]/[4]).  Same terms in
// the same order as k_cg_matvec (bit-identical results), organised by the
// lattice's 3 x 3 phases:
//  * tiles of 24 x 96 outputs start on lattice rows / columns (the host picks
//    the row offset of the slab's larger lattice-regular region), so in a
//    tile away from a periodic seam the lattice is every 3rd window row and
//    column;
//  * there every lane owns a 3-column triple and every warp a row triple:
//    the 3 x 3 lattice samples of a triple pair sit in registers and its 9
//    outputs contract them with compile-time tap indices (49 MACs, taps
//    warp-uniform, z reads conflict-free);
//  * tiles whose window crosses a seam (lattice spacing 1 or 2) take the
//    list-based path: lattice rows / columns compacted by warp ballots, each
//    output row / column building its <= 4 (sample, tap) pairs in parallel.
//  * a rank-one PSF (u v^T: the Gaussian of configs[2]/[4]) contracts both
//    stages as two 1-D passes in regular tiles: z = u * (v * w) at the
//    lattice, H^T z = u * (v * z) at the outputs -- 2.5x fewer shared loads,
//    1.6x fewer FMAs; the terms regrouped, equal to the 2-D sums to rounding.
constexpr int MVP_TH = 24, MVP_TW = 96, MVP_MAXL = 4;

struct MvpGeom {
  static constexpr int K = 7, S = 3, R = 3;
  static constexpr int HX = MVP_TH + 4 * R, WX = MVP_TW + 4 * R;  // w tile
  static constexpr int HZ = MVP_TH + 2 * R, WZ = MVP_TW + 2 * R;  // z_up window
  // lattice rows / columns in a window: spacing S except one periodic seam
  static constexpr int NZR = HZ / S + 2, NZC = WZ / S + 2;
  static constexpr int NLR = HZ / S, NLC = WZ / S;  // regular tiles
  static constexpr int KK = (K * K + 1) & ~1;       // taps, padded: the w tile 16-byte aligned
  static constexpr int HR = S * (NLR - 1) + K;      // window rows the lattice samples read
  static constexpr int NHS = HR * NLC > NLR * MVP_TW ? HR * NLC : NLR * MVP_TW;
  static constexpr int NINT = NZR + NZC + HZ + WZ + (MVP_TH + MVP_TW) * (MVP_MAXL + 1) + 4;
  // taps | w tile | z | rank-one passes | reduction scratch | index lists
  static constexpr size_t smem =
      sizeof(double) * ((size_t)KK + (size_t)HX * WX + (size_t)NZR * NZC + NHS + 64) +
      sizeof(int) * (size_t)NINT;
};

// output phase p (0..2) of a triple: its lattice samples d (0..2, ascending)
// and tap indices t; phase 0 uses all three, phases 1 / 2 the last two
__device__ __forceinline__ constexpr int mvp_tap(int p, int d) {
  return p == 0 ? 3 * d : (p == 1 ? 3 * d - 1 : 3 * d - 2);
}

// the shared-memory scratch of one tile's contraction
struct MvpSmem {
  const double* taps;
  double* zc;
  double* hs;  // rank-one PSF: row pass at the lattice columns, then the column pass
  int* ints;   // zr_pos | zc_pos | rcomp | ccomp | rlist | clist | nzr nzc irr
};

// i in [-n, 2n): periodic index without a division
__device__ __forceinline__ int wrap_near(int i, int n) {
  return i < 0 ? i + n : (i >= n ? i - n : i);
}

template <int MODE>
__device__ __forceinline__ bool mvp_vec_ok(const CgArgs& a, int j0) {
  using G = MvpGeom;
  return (a.W % 2) == 0 && j0 - 2 * G::R >= 0 && j0 - 2 * G::R + G::WX <= a.W;
}

// Synchronous tile load: 16-byte loads along interior rows, every thread's
// loads issued before its shared-memory stores (the load is the exposed latency)
template <int MODE>
__device__ __forceinline__ void mvp_load(const CgArgs& a, const double* src_x, const double* rr,
                                         const double* pold, bool cont, double beta, int i0,
                                         int j0, double* ws) {
  using G = MvpGeom;
  constexpr int R = G::R, HX = G::HX, WX = G::WX;
  const int H = a.H, W = a.W;
  if (mvp_vec_ok<MODE>(a, j0)) {
    constexpr int W2 = WX / 2, ITEMS = HX * W2, PER = (ITEMS + 255) / 256;
    double2 v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int it = threadIdx.x + 256 * q;
      const int ti = it / W2, c2 = it - ti * W2;
      v[q] = make_double2(0.0, 0.0);
      if (it < ITEMS) {
        const long long o = (long long)wrap_near(i0 - 2 * R + ti, H) * W + j0 - 2 * R + 2 * c2;
        if (MODE == CG_ITER) {
          const double2 rv = *reinterpret_cast<const double2*>(rr + o);
          if (cont) {
            const double2 pv = *reinterpret_cast<const double2*>(pold + o);
            v[q] = make_double2(fma(beta, pv.x, rv.x), fma(beta, pv.y, rv.y));
          } else {
            v[q] = rv;
          }
        } else {
          v[q] = *reinterpret_cast<const double2*>(src_x + o);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int it = threadIdx.x + 256 * q;
      if (it < ITEMS) *reinterpret_cast<double2*>(ws + 2 * it) = v[q];
    }
  } else {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int ti = warp; ti < HX; ti += 8) {
      const long long ro = (long long)wrap(i0 - 2 * R + ti, H) * W;
      for (int tj = lane; tj < WX; tj += 32) {
        const long long o = ro + wrap_fast(j0 - 2 * R + tj, W);
        double w;
        if (MODE == CG_ITER) w = cont ? fma(beta, pold[o], rr[o]) : rr[o];
        else w = src_x[o];
        ws[ti * WX + tj] = w;
      }
    }
  }
}

// Lattice of the tile's window (by GLOBAL row: a slab starts at global row
// a.row0 of an a.Hg-row image).  A tile (lattice-aligned origin) whose window
// crosses neither the buffer's wrap nor the global seam has the lattice on
// exactly the window rows / columns == 0 mod 3 (regular, decided in O(1));
// otherwise the lattice is compacted by ballots.  Ends on a barrier.
__device__ __forceinline__ bool mvp_regular(const CgArgs& a, int i0, int j0) {
  using G = MvpGeom;
  constexpr int R = G::R, S = G::S;
  const int lo = i0 - R, hi = i0 + G::HZ - R;  // window rows [lo, hi)
  if (lo < 0 || hi > a.H || j0 - R < 0 || j0 - R + G::WZ > a.W) return false;
  // a.seam: local row of global row 0 (-1: none); a.row0m = row0 mod Hg
  if (a.seam > lo && a.seam < hi) return false;
  const int g = (a.seam >= 0 && i0 >= a.seam) ? i0 - a.seam : a.row0m + i0;
  return g % S == 0;
}

__device__ __forceinline__ bool mvp_lattice(const CgArgs& a, int i0, int j0, const MvpSmem& m) {
  using G = MvpGeom;
  constexpr int R = G::R, S = G::S, HZ = G::HZ, WZ = G::WZ;
  if (mvp_regular(a, i0, j0)) {
    __syncthreads();
    return true;
  }
  int* zr_pos = m.ints;
  int* zc_pos = zr_pos + G::NZR;
  int* rcomp = zc_pos + G::NZC;
  int* ccomp = rcomp + HZ;
  int* sc = m.ints + G::NINT - 4;  // nzr, nzc, row irregular, column irregular
  const int H = a.H, W = a.W;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    int base = 0, irr = 0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int zi = c * 32 + lane;
      bool on = false;
      if (zi < HZ) {
        const int gu = wrap_fast(i0 - R + zi, H);
        const int gg = (a.Hg > 0) ? (int)(((long long)a.row0 + gu) % a.Hg) : gu;
        on = (gg % S) == 0;
        irr |= on != (zi % S == 0);
      }
      const unsigned msk = __ballot_sync(0xffffffffu, on);
      const int idx = base + __popc(msk & ((1u << lane) - 1u));
      if (zi < HZ) rcomp[zi] = on ? idx : -1;
      if (on) zr_pos[idx] = zi;
      base += __popc(msk);
    }
    irr = __any_sync(0xffffffffu, irr);
    if (lane == 0) {
      sc[0] = base;
      sc[2] = irr;
    }
  } else if (warp == 1) {
    int base = 0, irr = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int zj = c * 32 + lane;
      const bool on = zj < WZ && (wrap_fast(j0 - R + zj, W) % S) == 0;
      irr |= zj < WZ && on != (zj % S == 0);
      const unsigned msk = __ballot_sync(0xffffffffu, on);
      const int idx = base + __popc(msk & ((1u << lane) - 1u));
      if (zj < WZ) ccomp[zj] = on ? idx : -1;
      if (on) zc_pos[idx] = zj;
      base += __popc(msk);
    }
    irr = __any_sync(0xffffffffu, irr);
    if (lane == 0) {
      sc[1] = base;
      sc[3] = irr;
    }
  }
  __syncthreads();
  return (sc[2] | sc[3]) == 0;
}

// (H^T z_up)(u, v) of every output of the tile, handed to emit(oi, oj, ht).
// Starts after mvp_lattice's barrier with ws complete; ends with every read
// of ws / zc issued before the caller's next barrier.
template <class Emit>
__device__ __forceinline__ void mvp_contract(bool regular, const double* ws, const MvpSmem& m,
                                             const double* huv, Emit&& emit) {
  using G = MvpGeom;
  constexpr int K = G::K, S = G::S, R = G::R, WX = G::WX, NZC = G::NZC, NLC = G::NLC;
  constexpr int NLR = G::NLR, TH = MVP_TH, TW = MVP_TW, ML = MVP_MAXL;
  static_assert(G::HZ <= 64 && G::WZ <= 128, "ballot compaction covers 64 rows / 128 columns");
  static_assert(TH == 24 && TW == 96, "8 warps x a row triple, 32 lanes x a column triple");
  const double* taps = m.taps;
  double* zc = m.zc;
  int* zr_pos = m.ints;
  int* zc_pos = zr_pos + G::NZR;
  int* rcomp = zc_pos + NZC;
  int* ccomp = rcomp + G::HZ;
  int* rlist = ccomp + G::WZ;  // per output row: ML x (compact index << 8 | tap row), count
  int* clist = rlist + TH * (ML + 1);
  const int* sc = m.ints + G::NINT - 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (regular && huv) {
    double uu[K], vv[K];
#pragma unroll
    for (int t = 0; t < K; ++t) {
      uu[t] = __ldg(huv + t);
      vv[t] = __ldg(huv + K + t);
    }
    double* hs = m.hs;
    // h(row, lj) = sum_tb v[tb] w(row, 3 lj + 2r - tb)
    for (int idx = threadIdx.x; idx < G::HR * NLC; idx += blockDim.x) {
      const int row = idx / NLC, lj = idx - row * NLC;
      const double* wp = ws + row * WX + S * lj + 2 * R;
      double h = 0.0;
#pragma unroll
      for (int tb = 0; tb < K; ++tb) h = fma(vv[tb], wp[-tb], h);
      hs[idx] = h;
    }
    __syncthreads();
    // z(li, lj) = sum_ta u[ta] h(3 li + 2r - ta, lj)
    for (int idx = threadIdx.x; idx < NLR * NLC; idx += blockDim.x) {
      const int li = idx / NLC, lj = idx - li * NLC;
      const double* hp = hs + (S * li + 2 * R) * NLC + lj;
      double z = 0.0;
#pragma unroll
      for (int ta = 0; ta < K; ++ta) z = fma(uu[ta], hp[-ta * NLC], z);
      zc[idx] = z;
    }
    __syncthreads();
    // g(li, v) = sum_dc v[tap(pv, dc)] z(li, c + dc), v = 3 c + pv (into hs)
    for (int idx = threadIdx.x; idx < NLR * 32; idx += blockDim.x) {
      const int li = idx >> 5, c = idx & 31;
      double z3[3];
#pragma unroll
      for (int dc = 0; dc < 3; ++dc) z3[dc] = zc[li * NLC + c + dc];
#pragma unroll
      for (int pv = 0; pv < 3; ++pv) {
        double g = 0.0;
#pragma unroll
        for (int dc = pv == 0 ? 0 : 1; dc < 3; ++dc) g = fma(vv[mvp_tap(pv, dc)], z3[dc], g);
        hs[li * TW + 3 * c + pv] = g;
      }
    }
    __syncthreads();
    const int tr = warp;
#pragma unroll
    for (int pv = 0; pv < 3; ++pv) {
      double g3[3];
#pragma unroll
      for (int da = 0; da < 3; ++da) g3[da] = hs[(tr + da) * TW + 3 * lane + pv];
#pragma unroll
      for (int pu = 0; pu < 3; ++pu) {
        double ht = 0.0;
#pragma unroll
        for (int da = pu == 0 ? 0 : 1; da < 3; ++da) ht = fma(uu[mvp_tap(pu, da)], g3[da], ht);
        emit(3 * tr + pu, 3 * lane + pv, ht);
      }
    }
    return;
  }
  if (regular) {
    // z at lattice (li, lj) = window (3 li, 3 lj)
    for (int idx = threadIdx.x; idx < NLR * NLC; idx += blockDim.x) {
      const int li = idx / NLC, lj = idx - li * NLC;
      const double* wp = ws + (S * li + 2 * R) * WX + (S * lj + 2 * R);
      double z = 0.0;
#pragma unroll
      for (int ta = 0; ta < K; ++ta)
#pragma unroll
        for (int tb = 0; tb < K; ++tb) z = fma(taps[ta * K + tb], wp[-ta * WX - tb], z);
      zc[li * NLC + lj] = z;
    }
    __syncthreads();
    const int tr = warp;
    double z9[3][3];
#pragma unroll
    for (int da = 0; da < 3; ++da)
#pragma unroll
      for (int dc = 0; dc < 3; ++dc) z9[da][dc] = zc[(tr + da) * NLC + lane + dc];
#pragma unroll
    for (int pu = 0; pu < 3; ++pu)
#pragma unroll
      for (int pv = 0; pv < 3; ++pv) {
        double ht = 0.0;
#pragma unroll
        for (int da = pu == 0 ? 0 : 1; da < 3; ++da)
#pragma unroll
          for (int dc = pv == 0 ? 0 : 1; dc < 3; ++dc)
            ht = fma(taps[mvp_tap(pu, da) * K + mvp_tap(pv, dc)], z9[da][dc], ht);
        emit(3 * tr + pu, 3 * lane + pv, ht);
      }
    return;
  }
  const int nzr = sc[0], nzc = sc[1];
  // output row u (tile coords) reads window rows [u, u + 2r]; column v likewise
  if (threadIdx.x < TH) {
    const int u = threadIdx.x;
    int n = 0;
#pragma unroll
    for (int d = 0; d <= 2 * R; ++d) {
      const int c = rcomp[u + d];
      if (c >= 0 && n < ML) rlist[u * (ML + 1) + (n++)] = (c << 8) | d;
    }
    rlist[u * (ML + 1) + ML] = n;
  } else if (threadIdx.x >= 64 && threadIdx.x < 64 + TW) {
    const int v = threadIdx.x - 64;
    int n = 0;
#pragma unroll
    for (int d = 0; d <= 2 * R; ++d) {
      const int c = ccomp[v + d];
      if (c >= 0 && n < ML) clist[v * (ML + 1) + (n++)] = (c << 8) | d;
    }
    clist[v * (ML + 1) + ML] = n;
  }
  // z = H w at the lattice samples (taps in the order of k_cg_matvec)
  for (int idx = threadIdx.x; idx < nzr * nzc; idx += blockDim.x) {
    const int li = idx / nzc, lj = idx - li * nzc;
    const double* wp = ws + (zr_pos[li] + 2 * R) * WX + (zc_pos[lj] + 2 * R);
    double z = 0.0;
#pragma unroll
    for (int ta = 0; ta < K; ++ta)
#pragma unroll
      for (int tb = 0; tb < K; ++tb) z = fma(taps[ta * K + tb], wp[-ta * WX - tb], z);
    zc[li * NZC + lj] = z;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < TH * TW; idx += blockDim.x) {
    const int oi = idx / TW, oj = idx - oi * TW;
    const int* rl = rlist + oi * (ML + 1);
    const int* cl = clist + oj * (ML + 1);
    const int rn = rl[ML], cn = cl[ML];
    int ce[ML];
#pragma unroll
    for (int j = 0; j < ML; ++j) ce[j] = cl[j];
    double ht = 0.0;  // lattice rows then columns ascending
#pragma unroll
    for (int i = 0; i < ML; ++i) {
      if (i < rn) {
        const int re = rl[i];
        const double* trow = taps + (re & 255) * K;
        const double* zrow = zc + (re >> 8) * NZC;
#pragma unroll
        for (int j = 0; j < ML; ++j)
          if (j < cn) ht = fma(trow[ce[j] & 255], zrow[ce[j] >> 8], ht);
      }
    }
    emit(oi, oj, ht);
  }
}

__device__ __forceinline__ MvpSmem mvp_smem(double** ws) {
  using G = MvpGeom;
  double* base = reinterpret_cast<double*>(s_smem);
  *ws = base + G::KK;
  double* zc = *ws + G::HX * G::WX;
  double* hs = zc + G::NZR * G::NZC;
  return MvpSmem{base, zc, hs, reinterpret_cast<int*>(hs + G::NHS + 64)};
}

template <int MODE>
__global__ void __launch_bounds__(256, 4) k_cg_matvec_ct(CgArgs a) {
  using G = MvpGeom;
  constexpr int R = G::R, WX = G::WX, TH = MVP_TH, TW = MVP_TW;
  const int b = blockIdx.z;
  CgState& cs = a.cg[b];
  if (MODE == CG_INIT) {
    if (!takes_step(a.st[b], a.phase)) return;
  } else if (MODE == CG_ITER) {
    if (!cs.active) return;
  } else if (MODE == CG_RESID) {
    if (!takes_step(a.st[b], a.phase) || !cs.need_resid) return;
  }
  double* ws;
  const MvpSmem m = mvp_smem(&ws);
  double* taps = const_cast<double*>(m.taps);
  double* red = m.hs + G::NHS;
  for (int i = threadIdx.x; i < G::K * G::K; i += blockDim.x) taps[i] = a.taps[i];
  const int H = a.H, W = a.W;
  const long long N = (long long)H * W;
  const int i0 = a.tile_off + (blockIdx.y - 1) * TH, j0 = blockIdx.x * TW;
  const bool cont = MODE == CG_ITER && cs.its > 0;  // p = r + beta p_old after the 1st iteration
  const double beta = cont ? cs.beta : 0.0;
  const double* xin = (MODE == CG_ITER) ? nullptr : a.xin.at(b, a.st);
  mvp_load<MODE>(a, xin, a.r + (long long)b * N, a.p + (long long)b * N, cont, beta, i0, j0, ws);
  const bool regular = mvp_lattice(a, i0, j0, m);  // its barrier also completes ws
  double acc[2] = {0.0, 0.0};
  const double inv_s2 = a.inv_sigma2;
  mvp_contract(regular, ws, m, a.huv, [&](int oi, int oj, double ht) {
    const int gi = i0 + oi, gj = j0 + oj;
    if (gi < 0 || gi >= H || gj >= W) return;
    const double wv = ws[(oi + 2 * R) * WX + (oj + 2 * R)];
    const double aw = fma(ht, inv_s2, a.alpha * wv);
    const long long o = (long long)b * N + (long long)gi * W + gj;
    if (MODE == CG_PLAIN) {
      a.q[o] = aw;
    } else if (MODE == CG_ITER) {
      a.p[o] = wv;
      a.q[o] = aw;
      acc[0] = fma(wv, aw, acc[0]);
    } else {
      const double bb = fma(a.alpha, a.f[o], a.hty[o]);  // rhs = H^T y/sigma^2 + alpha f
      const double res = bb - aw;
      if (MODE == CG_INIT) {
        a.r[o] = res;
        a.xout.at(b, a.st)[(long long)gi * W + gj] = wv;  // warm start copy x <- x_k
      }
      acc[0] = fma(bb, bb, acc[0]);
      acc[1] = fma(res, res, acc[1]);
    }
  });
  if (MODE == CG_PLAIN) return;
  block_sum<2>(acc, red);
  const int nblk = gridDim.x * gridDim.y;
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0) {
    a.partials[((long long)b * nblk + blk) * 2] = acc[0];
    a.partials[((long long)b * nblk + blk) * 2 + 1] = acc[1];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double tt[2];
  if (lastb) gather_partials<2>(a.partials + (long long)b * nblk * 2, nblk, tt, red);
  if (lastb && threadIdx.x == 0) cg_reduce_finish<MODE>(cs, a, b, tt[0], tt[1]);
}

// Local row of a lattice-aligned tile origin: the lattice phase of the slab's
// larger regular region (before / after the global periodic seam).
static int mvp_tile_off(const CgArgs& a) {
  const int H = a.H;
  if (a.Hg <= 0) return 0;  // the buffer is the image: lattice rows 0, 3, ...
  const long long r0 = ((long long)a.row0 % a.Hg + a.Hg) % a.Hg;
  const int seam = (int)(a.Hg - r0);  // local row of global row 0
  const int before = (int)((3 - r0 % 3) % 3);
  if (seam <= 0 || seam >= H) return before;
  return (seam >= H - seam) ? before : seam % 3;
}

// x += alpha p ; r -= alpha q ; rho = r.r ; stopping decisions
__global__ void __launch_bounds__(256) k_cg_update(CgArgs a) {
  const int b = blockIdx.y;
  CgState& cs = a.cg[b];
  if (!cs.active) return;
  const long long N = (long long)a.H * a.W;
  const double al = cs.alpha;
  double* x = a.xout.at(b, a.st);
  double* r = a.r + (long long)b * N;
  const double* p = a.p + (long long)b * N;
  const double* q = a.q + (long long)b * N;
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    x[i] = fma(al, p[i], x[i]);
    const double rn = fma(-al, q[i], r[i]);
    r[i] = rn;
    acc[0] = fma(rn, rn, acc[0]);
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0) a.partials[(long long)b * nblk + blockIdx.x] = acc[0];
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double rr1[1];
  if (lastb) gather_partials<1>(a.partials + (long long)b * nblk, nblk, rr1, red);
  if (lastb && threadIdx.x == 0) {
    const double rho = rr1[0];
    const double rho_prev = cs.rho;
    cs.its += 1;
    if (cs.its >= a.maxiter) {  // loop exhausted: info = maxiter, no final test
      cs.active = 0;
      cs.info = a.maxiter;
      cs.need_resid = 1;
    } else if (sqrt(rho) < cs.atol) {
      cs.active = 0;
    }
    cs.beta = rho / rho_prev;
    cs.rho = rho;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.st[b].cg_its = cs.its;
}

// ||b|| == 0: scipy returns b itself (the zero vector)
__global__ void k_cg_zero_b(CgArgs a) {
  const int b = blockIdx.y;
  if (!takes_step(a.st[b], a.phase) || !a.cg[b].zero_b) return;
  const long long N = (long long)a.H * a.W;
  double* x = a.xout.at(b, a.st);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = 0.0;
}

// WHILE-node condition of the CG loop: another iteration while any image's
// CG is active (scipy's loop test, iterative.py:406, decided on the device)
__global__ void k_cg_continue(const CgState* cg, int B, cudaGraphConditionalHandle h) {
  int any = 0;
  for (int b = threadIdx.x; b < B; b += 32) any |= cg[b].active;
  any = __any_sync(0xffffffffu, any);
  if (threadIdx.x == 0) cudaGraphSetConditional(h, any ? 1u : 0u);
}
void launch_cg_continue(const CgArgs& a, cudaGraphConditionalHandle h, cudaStream_t s) {
  k_cg_continue<<<1, 32, 0, s>>>(a.cg, a.B, h);
}

size_t cg_matvec_smem(int k) {
  const int r = k / 2;
  return sizeof(double) * ((size_t)k * k + (size_t)(MV_TH + 4 * r) * (MV_TW + 4 * r) +
                           (size_t)(MV_TH + 2 * r) * (MV_TW + 2 * r) + 64) +
         sizeof(int) * ((size_t)(MV_TH + 2 * r) + (MV_TW + 2 * r) + 2 * MV_TH + 2 * MV_TW + 64);
}

// REDVE_MATVEC=generic: the runtime-(k, s) kernel for every operator (A/B tests)
static bool matvec_ct_ok(const CgArgs& a) {
  const char* e = getenv("REDVE_MATVEC");
  if (e && e[0] == 'g') return false;
  return a.k == 7 && a.factor == 3;
}

template <int MODE>
static void matvec_t(const CgArgs& a_in, cudaStream_t s) {
  if (matvec_ct_ok(a_in)) {
    CgArgs a = a_in;
    a.tile_off = mvp_tile_off(a);
    if (a.Hg > 0) {
      const long long r0 = ((long long)a.row0 % a.Hg + a.Hg) % a.Hg;
      const long long sm = (a.Hg - r0) % a.Hg;  // local row of global row 0
      a.row0m = (int)r0;
      a.seam = sm < a.H ? (int)sm : -1;
    } else {
      a.row0m = 0;
      a.seam = -1;
    }
    // tile rows start at tile_off - TH (the first covers rows [0, tile_off))
    const int ntx = cdivs(a.W, MVP_TW), nty = 1 + cdivs(a.H - a.tile_off, MVP_TH);
    static bool ct_done = false;
    if (!ct_done) {
      cudaFuncSetAttribute(k_cg_matvec_ct<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)MvpGeom::smem);
      ct_done = true;
    }
    k_cg_matvec_ct<MODE><<<dim3(ntx, nty, a.B), 256, MvpGeom::smem, s>>>(a);
    return;
  }
  const CgArgs& a = a_in;
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_cg_matvec<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    done = true;
  }
  dim3 grid(cdivs(a.W, MV_TW), cdivs(a.H, MV_TH), a.B);
  k_cg_matvec<MODE><<<grid, 256, cg_matvec_smem(a.k), s>>>(a);
}

int cg_matvec_blocks(int H, int W) {  // the larger of both kernels' tile counts
  const int g = cdivs(W, MV_TW) * cdivs(H, MV_TH);
  const int c = cdivs(W, MVP_TW) * (2 + cdivs(H, MVP_TH));
  return g > c ? g : c;
}
int cg_update_blocks(long long N) {
  int c = cdivs(N, 256 * 8);
  return c > 1184 ? 1184 : (c < 1 ? 1 : c);
}

void launch_cg_init(const CgArgs& a, cudaStream_t s) { matvec_t<CG_INIT>(a, s); }
void launch_cg_iter(const CgArgs& a, cudaStream_t s) { matvec_t<CG_ITER>(a, s); }
void launch_cg_resid(const CgArgs& a, cudaStream_t s) { matvec_t<CG_RESID>(a, s); }
void launch_normal_matvec(const CgArgs& a, cudaStream_t s) { matvec_t<CG_PLAIN>(a, s); }
void launch_cg_update(const CgArgs& a, cudaStream_t s) {
  k_cg_update<<<dim3(cg_update_blocks((long long)a.H * a.W), a.B), 256, 0, s>>>(a);
}
void launch_cg_zero_b(const CgArgs& a, cudaStream_t s) {
  k_cg_zero_b<<<dim3(cg_update_blocks((long long)a.H * a.W), a.B), 256, 0, s>>>(a);
}

// --------------------------------------------------------------- stencil denoisers into f
// f(x) for the CG route (the Fourier route fuses them into k_row_fwd).
__global__ void __launch_bounds__(256) k_denoise_view(View xin, DenoiseArgs dn, double* out,
                                                      const ImgState* st, int phase, int H, int W) {
  const int b = blockIdx.y;
  if (!takes_step(st[b], phase)) return;
  const long long N = (long long)H * W;
  const double* x = xin.at(b, st);
  double* o = out + (long long)b * N;
  const int r = dn.ksize / 2;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / W), j = (int)(idx - (long long)i * W);
    double v;
    if (dn.kind == DN_MEDIAN3) {
      double q[9];
      int n = 0;
      for (int a = -1; a <= 1; ++a)
        for (int c = -1; c <= 1; ++c) q[n++] = __ldg(x + (long long)wrap(i + a, H) * W + wrap(j + c, W));
      v = median9(q);
    } else if (dn.kind == DN_CONV) {
      v = 0.0;
      for (int a = 0; a < dn.ksize; ++a)
        for (int c = 0; c < dn.ksize; ++c)
          v = fma(dn.taps[a * dn.ksize + c],
                  __ldg(x + (long long)wrap(i - (a - r), H) * W + wrap(j - (c - r), W)), v);
    } else {
      v = x[idx];
    }
    o[idx] = v;
  }
}

void launch_denoise_view(View xin, DenoiseArgs dn, double* out, const ImgState* st, int phase,
                         int B, int H, int W, cudaStream_t s) {
  k_denoise_view<<<dim3(cg_update_blocks((long long)H * W), B), 256, 0, s>>>(xin, dn, out, st,
                                                                           phase, H, W);
}

// --------------------------------------------------------------- step record
// ||x+ - x||, ||x||, finiteness -> record_step (solvers.py:225-253)
__global__ void __launch_bounds__(256) k_step_record(RecordArgs a) {
  const int b = blockIdx.y;
  if (!takes_step(a.st[b], a.ctl.phase)) return;
  const double* xn = a.xnew.at(b, a.st);
  const double* xp = a.xprev.at(b, a.st);
  double acc[3] = {0.0, 0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.N;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = xn[i], u = xp[i], d = v - u;
    acc[0] = fma(d, d, acc[0]);
    acc[1] = fma(u, u, acc[1]);
    acc[2] += isfinite(v) ? 0.0 : 1.0;
  }
  __shared__ double red[96];
  block_sum<3>(acc, red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0)
    for (int i = 0; i < 3; ++i) a.partials[((long long)b * nblk + blockIdx.x) * 3 + i] = acc[i];
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double t[3];
  if (lastb) gather_partials<3>(a.partials + (long long)b * nblk * 3, nblk, t, red);
  if (lastb && threadIdx.x == 0) {
    record_step(a.st[b], b, t[0], t[1], t[2], a.S, a.ctl, a.tr);
    const int rec = a.st[b].k - 1;
    if (a.cg && a.tr.cg_iters && rec < a.tr.cap)
      a.tr.cg_iters[(long long)b * a.tr.cap + rec] = a.cg[b].its;
  }
}

void launch_step_record(const RecordArgs& a, int B, cudaStream_t s) {
  k_step_record<<<dim3(cg_update_blocks(a.N), B), 256, 0, s>>>(a);
}

}  // namespace redve
