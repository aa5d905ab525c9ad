// RED fixed-point / vector-extrapolation kernels for B200 (sm_100a), fp64.
//
// Fourier fixed-point step  x+ = x_b + IDFT( alpha/(d HW) * DFT f(x) ),
// d = |H^|^2/sigma^2 + alpha, x_b = IDFT(DFT(H^T y/sigma^2)/d)
// (objective.py:100-104; the split is exact algebra: the step is linear in
// its right-hand side).  Two images of the batch ride as one complex image
// (re = image 2p, im = image 2p+1): the spectral multiplier is real and
// even, so the complex transform of the pair yields both real results.
//
//   k_row_fwd : tile (+halo) -> fused denoiser -> row FFTs        -> Z
//   k_col     : Z columns -> FFT -> * alpha g -> inverse FFT        -> Z
//   k_row_inv : Z rows -> inverse FFT -> + x_b -> x+  (+ step-norm record)
//
// Per-image reductions are deterministic: per-CTA partials, then the last
// CTA of the image (atomic ticket) sums them in CTA order.
#include <cstdio>

#include "cost.cuh"
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace redve {

extern __shared__ __align__(16) unsigned char g_smem[];


static inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// --------------------------------------------------------------- setup
// Kernels that need more than 48 KB of dynamic shared memory raise their limit
// at first launch (next to the launch), so context creation only clears any
// stale error state.
int configure_kernels() {
  cudaGetLastError();
  return (int)cudaSuccess;
}

// raise a kernel's dynamic shared-memory limit to what the device allows
template <class K>
static cudaError_t allow_big_smem(K kernel, int optin) {
  if (optin < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kernel);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes);
}

__global__ void k_twiddles(cd* tw, int L) {
  int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < L) {
    double s, c;
    sincospi(2.0 * (double)m / (double)L, &s, &c);
    tw[m] = cd{c, s};
  }
}
void launch_twiddles(cd* tw, int L, cudaStream_t s) {
  k_twiddles<<<cdiv(L, 256), 256, 0, s>>>(tw, L);
}

// g[k1][k2] = 1 / ((|H^(k1,k2)|^2/sigma^2 + alpha) * H * W)   (objective.py:71-72)
// H^ = sum taps[a][b] exp(-2 pi i (k1 (a-r)/H + k2 (b-r)/W))   (imaging.py:113-129)
__global__ void k_inv_denom(double* g, int H, int W, const double* taps, int hk, double sigma,
                            double alpha) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= H * W) return;
  int k1 = idx / W, k2 = idx % W;
  int r = hk / 2;
  double re = 0.0, im = 0.0;
  for (int a = 0; a < hk; ++a) {
    long long pa = ((long long)k1 * (a - r)) % H;
    if (pa < 0) pa += H;
    for (int b = 0; b < hk; ++b) {
      long long pb = ((long long)k2 * (b - r)) % W;
      if (pb < 0) pb += W;
      double ph = (double)pa / H + (double)pb / W;  // in turns
      double s, c;
      sincospi(2.0 * ph, &s, &c);
      double t = taps[a * hk + b];
      re += t * c;
      im -= t * s;
    }
  }
  double d = (re * re + im * im) / (sigma * sigma) + alpha;
  g[idx] = 1.0 / (d * (double)H * (double)W);
}
void launch_inv_denom(double* g, int H, int W, const double* taps, int hk, double sigma,
                      double alpha, cudaStream_t s) {
  k_inv_denom<<<cdiv((long long)H * W, 128), 128, 0, s>>>(g, H, W, taps, hk, sigma, alpha);
}

static inline __host__ __device__ size_t al16(size_t b) { return (b + 15) & ~size_t(15); }

// --------------------------------------------------------------- cost
// E(x) = ||Hx - y||^2/(2 sigma^2) + alpha/2 x.(x - f(x))   (objective.py:78-88)
// PSNR = 10 log10(255^2 / mse)                          (imaging.py:234-248)
// Modes: record on the logging cadence (solvers.py:232-238, best-iterate
// tracking :235-236), note_initial (:219-223), finalize (:255-262).
template <int DK>
__global__ void __launch_bounds__(256) k_cost(CostArgs a) {
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < a.B;
  const bool w0 = cost_wants(a.st[b0], a);
  const bool w1 = has1 && cost_wants(a.st[b1], a);
  const int nblk = gridDim.x;
  if (!w0 && !w1) {
    // nothing to evaluate; block 0 still commits the step for stepped images
    if (a.mode == COST_RECORD && blockIdx.x == 0 && threadIdx.x == 0) {
      commit_step(a.st[b0], a.ctl.phase);
      if (has1) commit_step(a.st[b1], a.ctl.phase);
    }
    return;
  }
  const int W = a.W, H = a.H;
  const long long N = (long long)H * W;
  const int rH = a.hk / 2;
  const int Rd = DK == DN_CONV ? a.dn.ksize / 2 : (DK == DN_MEDIAN3 ? 1 : 0);
  const int R = max(rH, Rd);
  const int kk = DK == DN_CONV ? a.dn.ksize * a.dn.ksize : 0;
  double* s_h = reinterpret_cast<double*>(g_smem);
  double* s_taps = s_h + a.hk * a.hk + 2 * a.hk;
  double* s_red = s_taps + kk;
  cd* tile = reinterpret_cast<cd*>(
      g_smem + al16((a.hk * a.hk + 2 * a.hk + kk + 32 * 3 * 2) * sizeof(double)));
  cd* vbuf = tile + (size_t)(a.rows + 2 * R) * W;
  double* s_u = s_h + a.hk * a.hk;
  double* s_v = s_u + a.hk;
  for (int i = threadIdx.x; i < a.hk * a.hk; i += blockDim.x) s_h[i] = a.htaps[i];
  if (a.separable)
    for (int i = threadIdx.x; i < a.hk; i += blockDim.x) {
      s_u[i] = a.hu[i];
      s_v[i] = a.hv[i];
    }
  for (int i = threadIdx.x; i < kk; i += blockDim.x) s_taps[i] = a.dn.taps[i];
  const double* x0 = w0 ? a.x.at(b0, a.st) : nullptr;
  const double* x1 = w1 ? a.x.at(b1, a.st) : nullptr;
  const int r0 = blockIdx.x * a.rows;
  const int trows = a.rows + 2 * R;
  if ((W & 1) == 0) {
    const int W2 = W >> 1;
    for (int idx = threadIdx.x; idx < trows * W2; idx += blockDim.x) {
      const int i = idx / W2, c2 = idx - i * W2;
      const long long o = (long long)wrap(r0 - R + i, H) * W + 2 * c2;
      double2 u0 = x0 ? __ldg(reinterpret_cast<const double2*>(x0 + o)) : make_double2(0.0, 0.0);
      double2 u1 = x1 ? __ldg(reinterpret_cast<const double2*>(x1 + o)) : make_double2(0.0, 0.0);
      st_cd(tile + i * W + 2 * c2, cd{u0.x, u1.x});
      st_cd(tile + i * W + 2 * c2 + 1, cd{u0.y, u1.y});
    }
  } else {
    for (int idx = threadIdx.x; idx < trows * W; idx += blockDim.x) {
      const int i = idx / W, c = idx - i * W;
      const long long o = (long long)wrap(r0 - R + i, H) * W + c;
      st_cd(tile + idx, cd{x0 ? __ldg(x0 + o) : 0.0, x1 ? __ldg(x1 + o) : 0.0});
    }
  }
  __syncthreads();
  const int s = a.factor;
  if (a.separable) {  // vertical pass of the blur on the measurement-grid rows
    for (int idx = threadIdx.x; idx < a.rows * W; idx += blockDim.x) {
      const int li = idx / W, c = idx - li * W;
      const int row = r0 + li;
      if (row >= H || (row % s) != 0) continue;
      cd acc = cd{0.0, 0.0};
      for (int ta = 0; ta < a.hk; ++ta) {
        const cd xx = ld_cd(tile + (li + R - (ta - rH)) * W + c);
        acc.x = fma(s_u[ta], xx.x, acc.x);
        acc.y = fma(s_u[ta], xx.y, acc.y);
      }
      st_cd(vbuf + idx, acc);
    }
    __syncthreads();
  }
  double acc[6] = {0, 0, 0, 0, 0, 0};  // fid0, reg0, ssd0, fid1, reg1, ssd1
  for (int idx = threadIdx.x; idx < a.rows * W; idx += blockDim.x) {
    const int li = idx / W, c = idx - li * W;
    const int row = r0 + li;
    if (row >= H) break;
    const long long o = (long long)row * W + c;
    const cd xv = ld_cd(tile + (li + R) * W + c);
    cd fv;
    if (DK == DN_EXTERNAL) {
      fv = cd{x0 ? __ldg(a.fext + (long long)b0 * N + o) : 0.0,
              x1 ? __ldg(a.fext + (long long)b1 * N + o) : 0.0};
    } else {
      fv = denoise_at(tile, W, li + R, c, DK, a.dn.ksize, s_taps);
    }
    acc[1] = fma(xv.x, xv.x - fv.x, acc[1]);
    acc[4] = fma(xv.y, xv.y - fv.y, acc[4]);
    if (a.ref) {
      if (x0) {
        double d = xv.x - __ldg(a.ref + (long long)b0 * N + o);
        acc[2] = fma(d, d, acc[2]);
      }
      if (x1) {
        double d = xv.y - __ldg(a.ref + (long long)b1 * N + o);
        acc[5] = fma(d, d, acc[5]);
      }
    }
    if ((row % s) == 0 && (c % s) == 0) {
      // (H x)(row, c) = sum taps[a][b] x[row-(a-r), c-(b-r)], then - y
      cd hx = cd{0.0, 0.0};
      if (a.separable) {
        const cd* vr = vbuf + li * W;
        for (int tb = 0; tb < a.hk; ++tb) {
          const cd xx = ld_cd(vr + wrap(c - (tb - rH), W));
          hx.x = fma(s_v[tb], xx.x, hx.x);
          hx.y = fma(s_v[tb], xx.y, hx.y);
        }
      } else {
        for (int ta = 0; ta < a.hk; ++ta) {
          const cd* trow = tile + (li + R - (ta - rH)) * W;
          for (int tb = 0; tb < a.hk; ++tb) {
            const double w = s_h[ta * a.hk + tb];
            const cd xx = ld_cd(trow + wrap(c - (tb - rH), W));
            hx.x = fma(w, xx.x, hx.x);
            hx.y = fma(w, xx.y, hx.y);
          }
        }
      }
      const long long oy = (long long)(row / s) * a.Wy + (c / s);
      const long long Ny = (long long)a.Hy * a.Wy;
      if (x0) {
        double d = hx.x - __ldg(a.y + (long long)b0 * Ny + oy);
        acc[0] = fma(d, d, acc[0]);
      }
      if (x1) {
        double d = hx.y - __ldg(a.y + (long long)b1 * Ny + oy);
        acc[3] = fma(d, d, acc[3]);
      }
    }
  }
  block_sum<6>(acc, s_red);
  if (threadIdx.x == 0) {
    double* dst = a.partials + ((long long)p * nblk + blockIdx.x) * 6;
    for (int i = 0; i < 6; ++i) dst[i] = acc[i];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + p, nblk, &s_last);
  double tot[6];
  if (lastb) gather_partials<6>(a.partials + (long long)p * nblk * 6, nblk, tot, s_red);
  if (lastb && threadIdx.x == 0) {
    if (a.mode == COST_VALUE) {
      for (int i = 0; i < 3; ++i) {
        a.out_vals[b0 * 3 + i] = tot[i];
        if (has1) a.out_vals[b1 * 3 + i] = tot[3 + i];
      }
    } else {
      if (w0) cost_finish(a.st[b0], b0, tot[0], tot[1], tot[2], a.ref != nullptr, a);
      if (w1) cost_finish(a.st[b1], b1, tot[3], tot[4], tot[5], a.ref != nullptr, a);
    }
    if (a.mode == COST_RECORD) {
      commit_step(a.st[b0], a.ctl.phase);
      if (has1) commit_step(a.st[b1], a.ctl.phase);
    }
  }
}
int cost_rows(int H) { return H < 8 ? H : 8; }

// out[b] = ||y_b||^2, one CTA per image, fixed reduction order
__global__ void __launch_bounds__(256) k_sumsq(const double* y, long long n, double* out) {
  const double* yb = y + (long long)blockIdx.x * n;
  double acc[1] = {0.0};
  for (long long i = threadIdx.x; i < n; i += blockDim.x) acc[0] = fma(yb[i], yb[i], acc[0]);
  __shared__ double red[32];
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = acc[0];
}
void launch_sumsq(const double* y, long long n, int B, double* out, cudaStream_t s) {
  k_sumsq<<<B, 256, 0, s>>>(y, n, out);
}
template <int DK>
static void cost_t(const CostArgs& a, int npairs, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    allow_big_smem(k_cost<DK>, -1);
    done = true;
  }
  const int Rd = DK == DN_CONV ? a.dn.ksize / 2 : (DK == DN_MEDIAN3 ? 1 : 0);
  const int R = max(a.hk / 2, Rd);
  const int kk = DK == DN_CONV ? a.dn.ksize * a.dn.ksize : 0;
  size_t sm = al16((a.hk * a.hk + 2 * a.hk + kk + 32 * 3 * 2) * sizeof(double)) +
              (size_t)(a.rows + 2 * R) * a.W * sizeof(cd) +
              (a.separable ? (size_t)a.rows * a.W * sizeof(cd) : 0);
  dim3 grid(cdiv(a.H, a.rows), npairs);
  k_cost<DK><<<grid, 256, sm, s>>>(a);
}
void launch_cost(const CostArgs& a, int npairs, cudaStream_t s) {
  if (cost_fast_ok(a)) {
    launch_cost_fast(a, npairs, s);
    return;
  }
  switch (a.dn.kind) {
    case DN_CONV: cost_t<DN_CONV>(a, npairs, s); break;
    case DN_MEDIAN3: cost_t<DN_MEDIAN3>(a, npairs, s); break;
    case DN_EXTERNAL: cost_t<DN_EXTERNAL>(a, npairs, s); break;
    default: cost_t<DN_IDENTITY>(a, npairs, s); break;
  }
}

// --------------------------------------------------------------- copies
__global__ void k_copy_view(View dst, View src, int B, long long N, const ImgState* st,
                            int only_flag) {
  const int b = blockIdx.y;
  if (only_flag && !st[b].copy_best) return;
  double* d = dst.at(b, st);
  const double* s = src.at(b, st);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}
void launch_copy_view(View dst, View src, int B, long long N, const ImgState* st, int only_flag,
                      cudaStream_t s) {
  int chunks = cdiv(N, 256 * 8);
  if (chunks > 64) chunks = 64;
  k_copy_view<<<dim3(chunks, B), 256, 0, s>>>(dst, src, B, N, st, only_flag);
}

__global__ void k_gather(double* out, View cur, const double* best, int B, long long N,
                         const ImgState* st) {
  const int b = blockIdx.y;
  const double* s = st[b].use_best ? best + (long long)b * N : cur.at(b, st);
  double* d = out + (long long)b * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = s[i];
}
void launch_gather(double* out, View cur, const double* best, int B, long long N,
                   const ImgState* st, cudaStream_t s) {
  int chunks = cdiv(N, 256 * 8);
  if (chunks > 64) chunks = 64;
  k_gather<<<dim3(chunks, B), 256, 0, s>>>(out, cur, best, B, N, st);
}

// x0 into ring slot 0 (ring [B][S][N]) plus the reference's finiteness check of
// x0 (solvers.py:265-270, _as_vector) as a device flag: the solve graph does
// not depend on the caller's x0 pointer and no host sync precedes it.
__global__ void k_load_x0(double* ring, long long img_stride, const double* x0, int B, long long N,
                          int* bad) {
  const int b = blockIdx.y;
  const double* s = x0 + (long long)b * N;
  double* d = ring + (long long)b * img_stride;
  int nf = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = s[i];
    nf |= !isfinite(v);
    d[i] = v;
  }
  if (__syncthreads_or(nf) && threadIdx.x == 0) atomicOr(bad, 1);
}
void launch_load_x0(double* ring, long long img_stride, const double* x0, int B, long long N,
                    int* bad, cudaStream_t s) {
  int chunks = cdiv(N, 256 * 8);
  if (chunks > 64) chunks = 64;
  k_load_x0<<<dim3(chunks, B), 256, 0, s>>>(ring, img_stride, x0, B, N, bad);
}

__global__ void k_init_state(ImgState* st, int B) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ImgState s;
  memset(&s, 0, sizeof(s));
  s.best_cost = INFINITY;
  s.t0 = globaltimer_ns();
  st[b] = s;
}
void launch_init_state(ImgState* st, int B, cudaStream_t s) {
  k_init_state<<<cdiv(B, 128), 128, 0, s>>>(st, B);
}

// --------------------------------------------------------------- VE: Gram
__device__ __forceinline__ bool ve_participates(const ImgState& s) {
  return s.term == RUNNING || s.term == BUDGET;
}
__device__ __forceinline__ const double* slot_ptr(const VeArgs& a, int b, int slot) {
  return a.ring + (long long)b * a.img_stride + (long long)(slot % a.S) * a.slot_stride;
}

__device__ __noinline__ void mgs_block(const VeArgs& a, int b);

template <int KP1>
__global__ void __launch_bounds__(256) k_gram(VeArgs a) {
  constexpr int NG = KP1 * (KP1 + 1) / 2;
  const int b = blockIdx.y;
  ImgState& s = a.st[b];
  if (!ve_participates(s)) return;
  __shared__ double s_red[32 * NG];
  const double* w[KP1 + 1];
  const int s0 = s.start + a.m;
#pragma unroll
  for (int j = 0; j <= KP1; ++j) w[j] = slot_ptr(a, b, s0 + j);
  double acc[NG];
#pragma unroll
  for (int i = 0; i < NG; ++i) acc[i] = 0.0;
  // pairs of pixels with 16-byte loads (every slot starts 16-byte aligned when N is even)
  const long long N2 = (a.N & 1) ? 0 : (a.N >> 1);
#pragma unroll 2
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N2;
       p += (long long)gridDim.x * blockDim.x) {
    double d0[KP1], d1[KP1];
    double2 prev = __ldg(reinterpret_cast<const double2*>(w[0]) + p);
#pragma unroll
    for (int j = 0; j < KP1; ++j) {
      const double2 nx = __ldg(reinterpret_cast<const double2*>(w[j + 1]) + p);
      d0[j] = nx.x - prev.x;
      d1[j] = nx.y - prev.y;
      prev = nx;
    }
    int q = 0;
#pragma unroll
    for (int i = 0; i < KP1; ++i)
#pragma unroll
      for (int j = i; j < KP1; ++j) {
        acc[q] = fma(d0[i], d0[j], acc[q]);
        acc[q] = fma(d1[i], d1[j], acc[q]);
        ++q;
      }
  }
  for (long long p = 2 * N2 + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < a.N;
       p += (long long)gridDim.x * blockDim.x) {
    double d[KP1];
    double prev = __ldg(w[0] + p);
#pragma unroll
    for (int j = 0; j < KP1; ++j) {
      double nx = __ldg(w[j + 1] + p);
      d[j] = nx - prev;
      prev = nx;
    }
    int q = 0;
#pragma unroll
    for (int i = 0; i < KP1; ++i)
#pragma unroll
      for (int j = i; j < KP1; ++j) {
        acc[q] = fma(d[i], d[j], acc[q]);
        ++q;
      }
  }
  block_sum<NG>(acc, s_red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0) {
    double* dst = a.partials + ((long long)b * nblk + blockIdx.x) * NG;
    for (int i = 0; i < NG; ++i) dst[i] = acc[i];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double tot[NG];
  if (lastb) gather_partials<NG>(a.partials + (long long)b * nblk * NG, nblk, tot, s_red);
  if (lastb && threadIdx.x == 0) {
    double G[KP1 * KP1];
    int q = 0;
    for (int i = 0; i < KP1; ++i)
      for (int j = i; j < KP1; ++j) {
        G[i * KP1 + j] = tot[q];
        G[j * KP1 + i] = tot[q];
        ++q;
      }
    VeOut o;
    decide_from_gram(G, KP1, a.method, a.rank_tol, o);
    s.ve_mode = o.mode;
    if (o.mode == VE_EXTRAPOLATE) {
      s.ve_k = o.k_used;
      s.ve_method = o.method;
      s.ve_fallback = o.fallback;
      s.ve_stab = o.stab;
      for (int i = 0; i <= o.k_used; ++i) {
        s.ve_gamma[i] = o.gamma[i];
        s.ve_c[i] = o.c[i];
        if (i < o.k_used) s.ve_xi[i] = o.xi[i];
      }
    }
  }
  if (lastb && !a.mgs_cluster) {  // rank question below the Gram route's resolution: exact MGS
    __syncthreads();
    if (s.ve_mode == VE_MGS) mgs_block(a, b);
  }
}

template <int KP1>
static void launch_gram_t(const VeArgs& a, cudaStream_t s) {
  k_gram<KP1><<<dim3(a.chunks, a.B), 256, 0, s>>>(a);
}
void launch_gram(const VeArgs& a, cudaStream_t s) {
  switch (a.kp1) {
    case 2: launch_gram_t<2>(a, s); break;
    case 3: launch_gram_t<3>(a, s); break;
    case 4: launch_gram_t<4>(a, s); break;
    case 5: launch_gram_t<5>(a, s); break;
    case 6: launch_gram_t<6>(a, s); break;
    case 7: launch_gram_t<7>(a, s); break;
    case 8: launch_gram_t<8>(a, s); break;
    case 9: launch_gram_t<9>(a, s); break;
    case 10: launch_gram_t<10>(a, s); break;
    case 11: launch_gram_t<11>(a, s); break;
    default: launch_gram_t<12>(a, s); break;
  }
}

// --------------------------------------------------------------- VE: exact MGS route
// mgs_qr (extrapolation.py:159-196) for the rare windows whose rank question
// the Gram route cannot resolve.  One CTA per flagged image.
__device__ double block_dot(const double* u, const double* v, long long N, double* s_red) {
  double acc[1] = {0.0};
  for (long long p = threadIdx.x; p < N; p += blockDim.x) acc[0] = fma(u[p], v[p], acc[0]);
  block_sum<1>(acc, s_red);
  __shared__ double s_bc;
  if (threadIdx.x == 0) s_bc = acc[0];
  __syncthreads();
  return s_bc;
}

// The exact MGS route for image b by the whole calling block (any size):
// called by k_gram's last block for the windows its Gram route flagged.
__device__ __noinline__ void mgs_block(const VeArgs& a, int b) {
  ImgState& s = a.st[b];
  __shared__ double s_red[32];
  __shared__ double R[MAXKP1][MAXKP1];
  const int n = a.kp1;
  const long long N = a.N;
  double* Q = a.qscratch + (long long)b * n * N;
  if (threadIdx.x < MAXKP1 * MAXKP1) (&R[0][0])[threadIdx.x] = 0.0;
  __syncthreads();
  const int s0 = s.start + a.m;
  int rank = n;
  double r11 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double* xa = slot_ptr(a, b, s0 + i);
    const double* xb = slot_ptr(a, b, s0 + i + 1);
    double* qi = Q + (long long)i * N;
    for (long long p = threadIdx.x; p < N; p += blockDim.x) qi[p] = xb[p] - xa[p];
    __syncthreads();
    for (int sweep = 0; sweep < 2; ++sweep) {
      for (int j = 0; j < i; ++j) {
        const double* qj = Q + (long long)j * N;
        double proj = block_dot(qj, qi, N, s_red);
        if (threadIdx.x == 0) R[j][i] += proj;
        for (long long p = threadIdx.x; p < N; p += blockDim.x) qi[p] -= proj * qj[p];
        __syncthreads();
      }
    }
    double rii = sqrt(block_dot(qi, qi, N, s_red));
    if (threadIdx.x == 0) R[i][i] = rii;
    if (i == 0) {
      if (rii < 1e-300) {
        if (threadIdx.x == 0) s.ve_mode = VE_CONVERGED;
        return;
      }
      r11 = rii;
    } else if (rii < a.rank_tol * r11) {
      rank = i;
      break;
    }
    for (long long p = threadIdx.x; p < N; p += blockDim.x) qi[p] /= rii;
    __syncthreads();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bool finite = true;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) finite = finite && isfinite(R[i][j]);
    VeOut o;
    if (!finite) {
      o.mode = VE_SKIP;
    } else {
      decide_from_r(R, n, rank, a.method, o);
    }
    s.ve_mode = o.mode;
    if (o.mode == VE_EXTRAPOLATE) {
      s.ve_k = o.k_used;
      s.ve_method = o.method;
      s.ve_fallback = o.fallback;
      s.ve_stab = o.stab;
      for (int i = 0; i <= o.k_used; ++i) {
        s.ve_gamma[i] = o.gamma[i];
        s.ve_c[i] = o.c[i];
        if (i < o.k_used) s.ve_xi[i] = o.xi[i];
      }
    }
  }
}

// The same MGS with the window split across an 8-CTA cluster: each CTA owns a
// contiguous chunk of every column, projections and norms are reduced over
// the cluster through distributed shared memory in fixed rank order (every
// CTA forms the same R), so one window costs ~1/8 of the single-CTA route.
constexpr int MGS_CL = 8;

__global__ void __cluster_dims__(MGS_CL, 1, 1) __launch_bounds__(256)
    k_mgs_cluster(VeArgs a) {
  namespace cg = cooperative_groups;
  const int b = blockIdx.y;
  ImgState& s = a.st[b];
  if (!ve_participates(s) || s.ve_mode != VE_MGS) return;  // same in every CTA of the cluster
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  __shared__ double s_red[32];
  __shared__ double s_part[2];
  __shared__ double s_val;
  __shared__ double R[MAXKP1][MAXKP1];
  const int n = a.kp1;
  const long long N = a.N;
  const long long per = (N + MGS_CL - 1) / MGS_CL;
  const long long lo = rank * per, hi = lo + per < N ? lo + per : N;
  double* Q = a.qscratch + (long long)b * n * N;
  if (threadIdx.x < MAXKP1 * MAXKP1) (&R[0][0])[threadIdx.x] = 0.0;
  int parity = 0;
  // cluster-wide dot product of chunks, identical result in every CTA
  auto cdot = [&](const double* u, const double* v) -> double {
    double acc[1] = {0.0};
    for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) acc[0] = fma(u[p], v[p], acc[0]);
    block_sum<1>(acc, s_red);
    if (threadIdx.x == 0) s_part[parity] = acc[0];
    cluster.sync();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int r = 0; r < MGS_CL; ++r) t += cluster.map_shared_rank(s_part, r)[parity];
      s_val = t;
    }
    __syncthreads();
    parity ^= 1;
    return s_val;
  };
  const int s0 = s.start + a.m;
  int rank_e = n;
  double r11 = 0.0;
  bool stationary = false;
  for (int i = 0; i < n; ++i) {
    const double* xa = slot_ptr(a, b, s0 + i);
    const double* xb = slot_ptr(a, b, s0 + i + 1);
    double* qi = Q + (long long)i * N;
    for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) qi[p] = xb[p] - xa[p];
    __syncthreads();
    for (int sweep = 0; sweep < 2; ++sweep) {
      for (int j = 0; j < i; ++j) {
        const double* qj = Q + (long long)j * N;
        const double proj = cdot(qj, qi);
        if (threadIdx.x == 0) R[j][i] += proj;
        for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) qi[p] -= proj * qj[p];
        __syncthreads();
      }
    }
    const double rii = sqrt(cdot(qi, qi));
    if (threadIdx.x == 0) R[i][i] = rii;
    if (i == 0) {
      if (rii < 1e-300) {
        stationary = true;
        break;
      }
      r11 = rii;
    } else if (rii < a.rank_tol * r11) {
      rank_e = i;
      break;
    }
    for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) qi[p] /= rii;
    __syncthreads();
  }
  __syncthreads();
  if (rank == 0 && threadIdx.x == 0) {
    VeOut o;
    bool finite = true;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) finite = finite && isfinite(R[i][j]);
    if (stationary) o.mode = VE_CONVERGED;
    else if (!finite) o.mode = VE_SKIP;
    else decide_from_r(R, n, rank_e, a.method, o);
    s.ve_mode = o.mode;
    if (o.mode == VE_EXTRAPOLATE) {
      s.ve_k = o.k_used;
      s.ve_method = o.method;
      s.ve_fallback = o.fallback;
      s.ve_stab = o.stab;
      for (int i = 0; i <= o.k_used; ++i) {
        s.ve_gamma[i] = o.gamma[i];
        s.ve_c[i] = o.c[i];
        if (i < o.k_used) s.ve_xi[i] = o.xi[i];
      }
    }
  }
  cluster.sync();  // no CTA leaves while another may still read its s_part
}

bool mgs_cluster_pays(int B) { return B * MGS_CL <= 2 * 148; }

void launch_mgs_cluster(const VeArgs& a, cudaStream_t s) {
  k_mgs_cluster<<<dim3(MGS_CL, a.B), 256, 0, s>>>(a);
}

// --------------------------------------------------------------- VE: combine
// x = x_m + sum_{j<k} xi_j (x_{m+j+1} - x_{m+j})  written over the cycle-start
// slot; accepted only if finite (solvers.py:368-378).
template <int KE>
__device__ __forceinline__ double combine_span(const VeArgs& a, int b, int s0, double* out,
                                               const double* xi_s) {
  const double* w[KE + 1];
  double xi[KE];
#pragma unroll
  for (int j = 0; j <= KE; ++j) w[j] = slot_ptr(a, b, s0 + j);
#pragma unroll
  for (int j = 0; j < KE; ++j) xi[j] = xi_s[j];
  double nf = 0.0;
  const long long N2 = (a.N & 1) ? 0 : (a.N >> 1);
  // batches of U pixel pairs: every load of a batch is issued before its
  // stores (out is one of the window slots, so the compiler cannot hoist
  // loads across the stores by itself)
  constexpr int U = 4;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long p0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; p0 < N2; p0 += U * st) {
    double2 acc[U], prev[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long p = p0 + u * st;
      prev[u] = p < N2 ? reinterpret_cast<const double2*>(w[0])[p] : make_double2(0.0, 0.0);
      acc[u] = prev[u];
    }
#pragma unroll
    for (int j = 0; j < KE; ++j) {
      double2 nx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long p = p0 + u * st;
        nx[u] = p < N2 ? reinterpret_cast<const double2*>(w[j + 1])[p] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc[u].x = fma(xi[j], nx[u].x - prev[u].x, acc[u].x);
        acc[u].y = fma(xi[j], nx[u].y - prev[u].y, acc[u].y);
        prev[u] = nx[u];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long p = p0 + u * st;
      if (p < N2) {
        reinterpret_cast<double2*>(out)[p] = acc[u];
        nf += (isfinite(acc[u].x) ? 0.0 : 1.0) + (isfinite(acc[u].y) ? 0.0 : 1.0);
      }
    }
  }
  for (long long p = 2 * N2 + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < a.N;
       p += (long long)gridDim.x * blockDim.x) {
    double prev = w[0][p];
    double acc = prev;
#pragma unroll
    for (int j = 0; j < KE; ++j) {
      const double nx = w[j + 1][p];
      acc = fma(xi[j], nx - prev, acc);
      prev = nx;
    }
    out[p] = acc;
    nf += isfinite(acc) ? 0.0 : 1.0;
  }
  return nf;
}

template <int KP1>
__global__ void __launch_bounds__(256) k_combine(VeArgs a) {
  const int b = blockIdx.y;
  ImgState& s = a.st[b];
  if (!ve_participates(s)) return;
  const int mode = s.ve_mode;
  if (mode != VE_EXTRAPOLATE) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (mode == VE_CONVERGED && !a.stationary_continues) {
        s.cur = (s.start + a.m) % a.S;
        s.term = CONVERGED;
      }
      s.start = s.cur;
    }
    return;
  }
  __shared__ double s_xi[MAXKP1];
  __shared__ double s_red[32];
  const int ke = s.ve_k;
  // weights past the extrapolation order are zero: the span always walks the
  // full window (KP1 differences, compile-time) so the kernel's registers are
  // sized for this configuration, not for the largest kappa
  if (threadIdx.x < MAXKP1) s_xi[threadIdx.x] = threadIdx.x < ke ? s.ve_xi[threadIdx.x] : 0.0;
  __syncthreads();
  const int s0 = s.start + a.m;
  double* out = a.ring + (long long)b * a.img_stride + (long long)s.start * a.slot_stride;
  double nf[1];
  nf[0] = combine_span<KP1 - 1>(a, b, s0, out, s_xi);  // ke <= kappa = KP1 - 1
  block_sum<1>(nf, s_red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0) a.partials[(long long)b * nblk + blockIdx.x] = nf[0];
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double tot1[1];
  if (lastb) gather_partials<1>(a.partials + (long long)b * nblk, nblk, tot1, s_red);
  if (lastb && threadIdx.x == 0) {
    const double tot = tot1[0];
    if (tot == 0.0) {
      s.cur = s.start;
      const TraceBufs& tr = a.tr;
      if (s.k - 1 < tr.cap) tr.gamma[(long long)b * tr.cap + s.k - 1] = s.ve_stab;
      if (s.ncycles < tr.ccap) {
        long long c = (long long)b * tr.ccap + s.ncycles;
        tr.cyc_meta[c * 4 + 0] = s.ve_method;
        tr.cyc_meta[c * 4 + 1] = s.ve_fallback;
        tr.cyc_meta[c * 4 + 2] = ke;
        tr.cyc_meta[c * 4 + 3] = s.k - 1;
        tr.cyc_stab[c] = s.ve_stab;
        for (int i = 0; i < MAXKP1; ++i) {
          tr.cyc_gamma[c * MAXKP1 + i] = i <= ke ? s.ve_gamma[i] : 0.0;
          tr.cyc_c[c * MAXKP1 + i] = i <= ke ? s.ve_c[i] : 0.0;
        }
      }
      s.ncycles += 1;
    }
    // else: discard the cycle, continue from the last plain iterate (cur)
    s.start = s.cur;
  }
}
void launch_combine(const VeArgs& a, cudaStream_t s) {
  const dim3 grid(a.chunks, a.B);
  switch (a.kp1) {
#define COMBINE_CASE(K) \
  case K: k_combine<K><<<grid, 256, 0, s>>>(a); break;
    COMBINE_CASE(2) COMBINE_CASE(3) COMBINE_CASE(4) COMBINE_CASE(5) COMBINE_CASE(6)
    COMBINE_CASE(7) COMBINE_CASE(8) COMBINE_CASE(9) COMBINE_CASE(10) COMBINE_CASE(11)
#undef COMBINE_CASE
    default: k_combine<12><<<grid, 256, 0, s>>>(a); break;
  }
}

// Pair-per-thread streaming stencils (even W): the (row, pair) position is
// advanced incrementally, neighbours come from L1, 16-byte stores.
static int pair_chunks(int B, long long N) {
  int c = (int)((1184 + B - 1) / B);
  const long long per = (N / 2 + 255) / 256;
  if (c > per) c = (int)per;
  if (c > 1024) c = 1024;
  return c < 1 ? 1 : c;
}

template <int MODE>  // 0: 3x3 median, 1: k x k stencil (corr / conv, scaled)
__global__ void __launch_bounds__(256) k_pairs(const double* __restrict__ x,
                                               double* __restrict__ out, int H, int W,
                                               const double* taps, int k, int corr,
                                               double scale) {
  const long long N = (long long)H * W;
  const int b = blockIdx.y;
  const double* __restrict__ xb = x + (long long)b * N;
  double* __restrict__ ob = out + (long long)b * N;
  const int W2 = W >> 1;
  const long long P = N >> 1;
  const long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int di = (int)(stride / W2), dj = (int)(stride % W2);
  int i = (int)(q0 / W2), j2 = (int)(q0 % W2);
  DenoiseArgs dn{DN_MEDIAN3, 0, 1, nullptr};
  // out never aliases x (operator / denoiser API contract), so unrolled
  // iterations' loads may issue ahead of the previous stores
#pragma unroll 4
  for (long long q = q0; q < P; q += stride) {
    const int j = 2 * j2;
    double f0, f1;
    if (MODE == 0) {
      fk_pair<DN_MEDIAN3>(xb, H, W, i, j, dn, nullptr, f0, f1);
    } else {
      stencil_pair(xb, H, W, i, j, taps, k, corr, f0, f1);
      f0 *= scale;
      f1 *= scale;
    }
    *reinterpret_cast<double2*>(ob + (long long)i * W + j) = make_double2(f0, f1);
    i += di;
    j2 += dj;
    if (j2 >= W2) {
      j2 -= W2;
      ++i;
    }
  }
}

// Eight outputs per thread along a row (W % 8 == 0): each tap row is read once
// as a register window of 8 + K - 1 values (L1/L2), the 8 accumulators share
// it, the stores are 16-byte.  Same taps and summation order as k_conv, so
// results are identical; the median shares sorted columns across the 8.
static int seg_chunks(int B, long long segs) {
  int c = (int)((1184 + B - 1) / B);
  const long long per = (segs + 255) / 256;
  if (c > per) c = (int)per;
  if (c > 1024) c = 1024;
  return c < 1 ? 1 : c;
}

template <int K, int CORR>
__global__ void __launch_bounds__(256) k_stencil8(const double* x, double* out, int H, int W,
                                                  const double* taps, double scale) {
  constexpr int R = K / 2, WIN = 8 + K - 1;
  __shared__ double s_t[K * K];
  for (int q = threadIdx.x; q < K * K; q += blockDim.x) s_t[q] = taps[q];
  __syncthreads();
  const long long N = (long long)H * W;
  const int b = blockIdx.y;
  const double* xb = x + (long long)b * N;
  double* ob = out + (long long)b * N;
  const int S8 = W >> 3;
  const long long P = (long long)H * S8;
  const long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const int di = (int)(stride / S8), ds = (int)(stride % S8);
  int i = (int)(q0 / S8), sg = (int)(q0 % S8);
  for (long long q = q0; q < P; q += stride) {
    const int j0 = 8 * sg;
    const bool inner = j0 - R >= 0 && j0 + 7 + R < W;
    double acc[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) acc[m] = 0.0;
#pragma unroll
    for (int ta = 0; ta < K; ++ta) {
      const int da = CORR ? (ta - R) : (R - ta);
      const double* row = xb + (long long)wrap_fast(i + da, H) * W;
      double w[WIN];
      if (inner) {
#pragma unroll
        for (int u = 0; u < WIN; ++u) w[u] = __ldg(row + j0 - R + u);
      } else {
#pragma unroll
        for (int u = 0; u < WIN; ++u) w[u] = __ldg(row + wrap_fast(j0 - R + u, W));
      }
#pragma unroll
      for (int tb = 0; tb < K; ++tb) {
        const double t = s_t[ta * K + tb];
#pragma unroll
        for (int m = 0; m < 8; ++m) acc[m] = fma(t, w[CORR ? m + tb : m + K - 1 - tb], acc[m]);
      }
    }
    double2* o2 = reinterpret_cast<double2*>(ob + (long long)i * W + j0);
#pragma unroll
    for (int m = 0; m < 4; ++m) o2[m] = make_double2(scale * acc[2 * m], scale * acc[2 * m + 1]);
    i += di;
    sg += ds;
    if (sg >= S8) {
      sg -= S8;
      ++i;
    }
  }
}

// Standalone 3x3 median, column-walking: each lane owns one image column and
// walks down MR rows, loading one new (coalesced) value per output and
// keeping the sorted 3-row column in registers; neighbours' sorted columns
// come by warp shuffles.  A warp yields 30 outputs (lanes 0 and 31 are the
// horizontal halo), so every input byte is read ~1.07x and the only traffic
// is the image in and f out.
constexpr int MR = 32;

__global__ void __launch_bounds__(128) k_median_cols(const double* __restrict__ x,
                                                     double* __restrict__ out, int H, int W) {
  const long long N = (long long)H * W;
  const int b = blockIdx.z;
  const double* __restrict__ xb = x + (long long)b * N;
  double* __restrict__ ob = out + (long long)b * N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c_out0 = (blockIdx.x * 4 + warp) * 30;  // first output column of this warp
  const int c = wrap_fast(c_out0 - 1 + lane, W);    // this lane's column
  const bool emits = lane >= 1 && lane <= 30 && c_out0 - 1 + lane < W;
  const int r0 = blockIdx.y * MR;
  const int rend = min(r0 + MR, H);
  double a = __ldg(xb + (long long)wrap_fast(r0 - 1, H) * W + c);
  double m = __ldg(xb + (long long)r0 * W + c);
  // batches of 8 rows: the 8 loads issue before the first median of the batch
  // (the shuffles keep the compiler from hoisting them by itself)
  for (int ib = r0; ib < rend; ib += 8) {
    double nx[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      nx[u] = ib + u < rend ? __ldg(xb + (long long)wrap_fast(ib + u + 1, H) * W + c) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (ib + u >= rend) break;
      const double e = nx[u];
      double lo = a, mi = m, hi = e;
      sort2(lo, mi);
      sort2(mi, hi);
      sort2(lo, mi);
      const double llo = __shfl_up_sync(0xffffffffu, lo, 1),
                   lmi = __shfl_up_sync(0xffffffffu, mi, 1),
                   lhi = __shfl_up_sync(0xffffffffu, hi, 1);
      const double rlo = __shfl_down_sync(0xffffffffu, lo, 1),
                   rmi = __shfl_down_sync(0xffffffffu, mi, 1),
                   rhi = __shfl_down_sync(0xffffffffu, hi, 1);
      if (emits)
        ob[(long long)(ib + u) * W + c] = med3d(dmax(dmax(llo, lo), rlo), med3d(lmi, mi, rmi),
                                                dmin(dmin(lhi, hi), rhi));
      a = m;
      m = e;
    }
  }
}

static bool launch_median_cols(const double* x, double* out, int B, int H, int W, cudaStream_t s) {
  if (W < 3 || H < 2) return false;
  dim3 grid((W + 119) / 120, (H + MR - 1) / MR, B);
  k_median_cols<<<grid, 128, 0, s>>>(x, out, H, W);
  return true;
}

template <int K>
static bool stencil8_k(const double* x, double* out, int B, int H, int W, const double* taps,
                       int corr, double scale, cudaStream_t s) {
  const dim3 grid(seg_chunks(B, (long long)H * (W / 8)), B);
  if (corr) k_stencil8<K, 1><<<grid, 256, 0, s>>>(x, out, H, W, taps, scale);
  else k_stencil8<K, 0><<<grid, 256, 0, s>>>(x, out, H, W, taps, scale);
  return true;
}

static bool launch_stencil8(const double* x, double* out, int B, int H, int W, const double* taps,
                            int k, int corr, double scale, cudaStream_t s) {
  if (W % 8 != 0 || W < 8 + k) return false;
  switch (k) {
    case 3: return stencil8_k<3>(x, out, B, H, W, taps, corr, scale, s);
    case 5: return stencil8_k<5>(x, out, B, H, W, taps, corr, scale, s);
    case 7: return stencil8_k<7>(x, out, B, H, W, taps, corr, scale, s);
    case 9: return stencil8_k<9>(x, out, B, H, W, taps, corr, scale, s);
    default: return false;
  }
}

// Rank-one K x K stencil (taps = u v^T: the uniform and Gaussian PSFs) as two
// 1-D passes over a shared-memory tile: 2K FMAs per output instead of K^2 and
// every input read once from HBM.  out = scale * (conv or corr)(x), periodic.
// The terms are regrouped: equal to the 2-D sum to rounding.
constexpr int SEP_TH = 32, SEP_TW = 64;

template <int K, int CORR>
__global__ void __launch_bounds__(256) k_sep_stencil(const double* x, double* out, int H, int W,
                                                     const double* uv, double scale) {
  constexpr int XW = SEP_TW + K - 1, XH = SEP_TH + K - 1, R = K / 2;
  __shared__ double xs[XH][XW];
  __shared__ double hs[XH][SEP_TW];
  const int b = blockIdx.z;
  const long long N = (long long)H * W;
  const double* xb = x + (long long)b * N;
  const int i0 = blockIdx.y * SEP_TH, j0 = blockIdx.x * SEP_TW;
  for (int idx = threadIdx.x; idx < XH * XW; idx += blockDim.x) {
    const int r = idx / XW, c = idx - r * XW;
    xs[r][c] = __ldg(xb + (long long)wrap_fast(i0 - R + r, H) * W + wrap_fast(j0 - R + c, W));
  }
  double u[K], v[K];
#pragma unroll
  for (int t = 0; t < K; ++t) {
    u[t] = __ldg(uv + t);
    v[t] = __ldg(uv + K + t);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < XH * SEP_TW; idx += blockDim.x) {
    const int r = idx / SEP_TW, c = idx - r * SEP_TW;
    double h = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) h = fma(v[t], xs[r][CORR ? c + t : c + K - 1 - t], h);
    hs[r][c] = h;
  }
  __syncthreads();
  double* ob = out + (long long)b * N;
  for (int idx = threadIdx.x; idx < SEP_TH * SEP_TW; idx += blockDim.x) {
    const int r = idx / SEP_TW, c = idx - r * SEP_TW;
    const int gi = i0 + r, gj = j0 + c;
    if (gi >= H || gj >= W) continue;
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < K; ++t) acc = fma(u[t], hs[CORR ? r + t : r + K - 1 - t][c], acc);
    ob[(long long)gi * W + gj] = scale * acc;
  }
}

template <int K>
static void sep_k(const double* x, double* out, int B, int H, int W, const double* uv, int corr,
                  double scale, cudaStream_t s) {
  const dim3 grid(cdiv(W, SEP_TW), cdiv(H, SEP_TH), B);
  if (corr) k_sep_stencil<K, 1><<<grid, 256, 0, s>>>(x, out, H, W, uv, scale);
  else k_sep_stencil<K, 0><<<grid, 256, 0, s>>>(x, out, H, W, uv, scale);
}

bool launch_conv_rank1(const double* x, double* out, int B, int H, int W, const double* uv, int k,
                       int corr, double scale, cudaStream_t s) {
  if (H < k || W < k) return false;
  switch (k) {
    case 3: sep_k<3>(x, out, B, H, W, uv, corr, scale, s); return true;
    case 5: sep_k<5>(x, out, B, H, W, uv, corr, scale, s); return true;
    case 7: sep_k<7>(x, out, B, H, W, uv, corr, scale, s); return true;
    case 9: sep_k<9>(x, out, B, H, W, uv, corr, scale, s); return true;
    default: return false;
  }
}

// --------------------------------------------------------------- stencils (operator API)
// out = scale * (conv or corr)(x, taps), periodic   (imaging.py:132-170)
__global__ void k_conv(const double* x, double* out, int B, int H, int W, const double* taps,
                       int k, int corr, double scale) {
  const long long N = (long long)H * W;
  const int r = k / 2;
  const int b = blockIdx.y;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx / W), j = (int)(idx - (long long)i * W);
    double acc = 0.0;
    for (int a = 0; a < k; ++a)
      for (int c = 0; c < k; ++c) {
        int di = corr ? (a - r) : -(a - r);
        int dj = corr ? (c - r) : -(c - r);
        acc = fma(taps[a * k + c], __ldg(x + (long long)b * N + (long long)wrap(i + di, H) * W +
                                             wrap(j + dj, W)),
                  acc);
      }
    out[(long long)b * N + idx] = scale * acc;
  }
}
void launch_conv(const double* x, double* out, int B, int H, int W, const double* taps, int k,
                 int corr, double scale, cudaStream_t s) {
  long long N = (long long)H * W;
  if (launch_stencil8(x, out, B, H, W, taps, k, corr, scale, s)) return;
  if ((W & 1) == 0 && W >= 2) {
    k_pairs<1><<<dim3(pair_chunks(B, N), B), 256, 0, s>>>(x, out, H, W, taps, k, corr, scale);
    return;
  }
  int chunks = cdiv(N, 256);
  if (chunks > 1024) chunks = 1024;
  k_conv<<<dim3(chunks, B), 256, 0, s>>>(x, out, B, H, W, taps, k, corr, scale);
}

// BlurDownsample.apply: conv, keep indices == 0 mod s   (imaging.py:193-197)
__global__ void k_decimate_conv(const double* x, double* out, int B, int H, int W, int f,
                                const double* taps, int k) {
  const int Hy = (H + f - 1) / f, Wy = (W + f - 1) / f;
  const long long Ny = (long long)Hy * Wy, N = (long long)H * W;
  const int r = k / 2, b = blockIdx.y;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < Ny;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx / Wy) * f, j = (int)(idx % Wy) * f;
    double acc = 0.0;
    for (int a = 0; a < k; ++a)
      for (int c = 0; c < k; ++c)
        acc = fma(taps[a * k + c],
                  __ldg(x + (long long)b * N + (long long)wrap(i - (a - r), H) * W +
                        wrap(j - (c - r), W)),
                  acc);
    out[(long long)b * Ny + idx] = acc;
  }
}
void launch_decimate_conv(const double* x, double* out, int B, int H, int W, int factor,
                          const double* taps, int k, cudaStream_t s) {
  long long Ny = (long long)((H + factor - 1) / factor) * ((W + factor - 1) / factor);
  int chunks = cdiv(Ny, 256);
  if (chunks > 1024) chunks = 1024;
  k_decimate_conv<<<dim3(chunks, B), 256, 0, s>>>(x, out, B, H, W, factor, taps, k);
}

// BlurDownsample.adjoint: zero-fill then correlate   (imaging.py:199-204)
__global__ void k_upsample_corr(const double* z, double* out, int B, int H, int W, int f,
                                const double* taps, int k, double scale) {
  const int Hy = (H + f - 1) / f, Wy = (W + f - 1) / f;
  const long long Ny = (long long)Hy * Wy, N = (long long)H * W;
  const int r = k / 2, b = blockIdx.y;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx / W), j = (int)(idx - (long long)i * W);
    double acc = 0.0;
    for (int a = 0; a < k; ++a) {
      int u = wrap(i + (a - r), H);
      if (u % f) continue;
      for (int c = 0; c < k; ++c) {
        int v = wrap(j + (c - r), W);
        if (v % f) continue;
        acc = fma(taps[a * k + c], __ldg(z + (long long)b * Ny + (long long)(u / f) * Wy + v / f),
                  acc);
      }
    }
    out[(long long)b * N + idx] = scale * acc;
  }
}
void launch_upsample_corr(const double* z, double* out, int B, int H, int W, int factor,
                          const double* taps, int k, double scale, cudaStream_t s) {
  long long N = (long long)H * W;
  int chunks = cdiv(N, 256);
  if (chunks > 1024) chunks = 1024;
  k_upsample_corr<<<dim3(chunks, B), 256, 0, s>>>(z, out, B, H, W, factor, taps, k, scale);
}

__global__ void k_median3(const double* x, double* out, int B, int H, int W) {
  const long long N = (long long)H * W;
  const int b = blockIdx.y;
  const double* xb = x + (long long)b * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    int i = (int)(idx / W), j = (int)(idx - (long long)i * W);
    double v[9];
    int q = 0;
    for (int a = -1; a <= 1; ++a)
      for (int c = -1; c <= 1; ++c)
        v[q++] = __ldg(xb + (long long)wrap(i + a, H) * W + wrap(j + c, W));
    out[(long long)b * N + idx] = median9(v);
  }
}
void launch_median3(const double* x, double* out, int B, int H, int W, cudaStream_t s) {
  long long N = (long long)H * W;
  if (launch_median_cols(x, out, B, H, W, s)) return;
  if ((W & 1) == 0 && W >= 4) {
    k_pairs<0><<<dim3(pair_chunks(B, N), B), 256, 0, s>>>(x, out, H, W, nullptr, 3, 0, 1.0);
    return;
  }
  int chunks = cdiv(N, 256);
  if (chunks > 1024) chunks = 1024;
  k_median3<<<dim3(chunks, B), 256, 0, s>>>(x, out, B, H, W);
}

}  // namespace redve

namespace redve {
// window-level extrapolate_once: the window is a ring of `S` = kappa+2 slots,
// cycle start at slot 0, current iterate = last row.
__global__ void k_window_setup(ImgState* st, int B, int S, int m) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  st[b].start = 0;
  st[b].cur = S - 1;
  st[b].k = 1;
  st[b].term = RUNNING;
  (void)m;
}
void launch_window_extrapolate_setup(ImgState* st, int B, int S, int m, cudaStream_t s) {
  k_window_setup<<<cdiv(B, 128), 128, 0, s>>>(st, B, S, m);
}
}  // namespace redve
