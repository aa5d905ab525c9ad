// Fused Fourier fixed-point step for circulant H (objective.py:100-104), fp64.
//
//   x+ = x_b + IDFT( alpha g . DFT f(x) ),  g = 1/((|H^|^2/sigma^2 + alpha) H W)
//   x_b = IDFT( g . DFT(H^T y / sigma^2) )            (precomputed once)
//
// The step is linear in its right-hand side, so splitting off x_b is exact
// algebra.  Two images of the batch ride as one complex image (re = 2p,
// im = 2p+1): g is real and even, so the complex transform of the pair gives
// both real results.  Three kernels per step, each streaming HBM once:
//
//   k_row_fwd : x tile (+halo) -> denoiser -> row FFTs            -> Z   (2 B N s)
//   k_col     : Z columns -> FFT -> * alpha g -> inverse FFT       -> Z   (2 B N s)
//   k_row_inv : Z rows -> inverse FFT -> + x_b -> x+, step-norm record    (4 B N s)
//
// Sizes that are powers of two in [16, 1024] use compile-time FFT plans;
// anything else the runtime plan (direct DFT for non powers of two).
#include "cost.cuh"
#include "kernels.cuh"

namespace redve {

extern __shared__ __align__(16) unsigned char f_smem[];

static inline __host__ __device__ size_t al16f(size_t b) { return (b + 15) & ~size_t(15); }
static inline int cdivf(long long a, long long b) { return (int)((a + b - 1) / b); }

static bool ct_size(int L) { return L == 64 || L == 128 || L == 256 || L == 512 || L == 1024; }
static size_t tw_bytes(int L) { return al16f((ct_size(L) ? tw_stage_size(L) : L) * sizeof(cd)); }

size_t row_fwd_smem(int W, int lpc, int radius, int ksize) {
  size_t tile = (size_t)(lpc + 2 * radius) * RowLayout::stride_for(W) * sizeof(cd);
  size_t lines = (size_t)lpc * RowLayout::stride_for(W) * sizeof(cd);
  return tw_bytes(W) + al16f((size_t)ksize * ksize * sizeof(double)) +
         (tile > lines ? tile : lines);
}
size_t col_smem(int H, int lpc) {
  const int T = threads_per_line(H);
  return tw_bytes(H) + (size_t)H * lpc * sizeof(cd) + (size_t)16 * T * lpc * sizeof(double);
}
size_t row_inv_smem(int W, int lpc) {
  return tw_bytes(W) + (size_t)lpc * RowLayout::stride_for(W) * sizeof(cd) +
         al16f(32 * 6 * sizeof(double));
}

__global__ void k_stage_twiddles(cd* tws, int L) {
  // stage (NS, R): tws[off + r*NS + k] = exp(2 pi i r k / (NS R))
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  int ns = 16, rem = L / 16, off = 0;
  while (rem > 1) {
    const int R = rem >= 16 ? 16 : rem;
    if (idx >= off && idx < off + R * ns) {
      const int e = idx - off, r = e / ns, k = e - r * ns;
      double s, c;
      sincospi(2.0 * (double)(r * k) / (double)(ns * R), &s, &c);
      tws[idx] = cd{c, s};
      return;
    }
    off += R * ns;
    ns *= R;
    rem /= R;
  }
}
void launch_stage_twiddles(cd* tws, int L, cudaStream_t s) {
  const int n = tw_stage_size(L);
  k_stage_twiddles<<<cdivf(n, 256), 256, 0, s>>>(tws, L);
}

template <int L, bool INV, class Lay>
__device__ __forceinline__ void fft_dispatch(cd (&v)[16], cd* sm, const cd* tw, int Lrt, int t,
                                             int line, const Lay& lay) {
  if constexpr (L > 0) {
    line_fft_ct<L, INV>(v, sm, tw, t, line, lay);
  } else {
    line_fft<INV>(v, sm, tw, Lrt, t, line, lay);
  }
}

// --------------------------------------------------------------- row forward
template <int LW>
__device__ __forceinline__ int colwrap(int c, int W) {
  if constexpr (LW > 0) return edge_wrap(c, W);  // |c - [0,W)| <= radius
  else return wrap(c, W);
}

constexpr int RF_BATCH = 10;

template <int LW, int DK>
__global__ void __launch_bounds__(256) k_row_fwd(RowFwdArgs a) {
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const bool a0 = takes_step(a.st[b0], a.phase);
  const bool a1 = b1 < a.B && takes_step(a.st[b1], a.phase);
  if (!a0 && !a1) return;
  const int W = LW > 0 ? LW : a.W;
  const int H = a.H;
  const int T = LW > 0 ? LW / 16 : threads_per_line(W);
  const int R = DK == DN_CONV ? a.dn.ksize / 2 : (DK == DN_MEDIAN3 ? 1 : 0);
  const int ks = DK == DN_CONV ? a.dn.ksize : 0;
  const int ntw = LW > 0 ? tw_stage_size(LW) : W;
  cd* s_tw = reinterpret_cast<cd*>(f_smem);
  double* s_taps = reinterpret_cast<double*>(f_smem + al16f(ntw * sizeof(cd)));
  cd* s_work = reinterpret_cast<cd*>(f_smem + al16f(ntw * sizeof(cd)) +
                                     al16f((size_t)a.dn.ksize * a.dn.ksize * sizeof(double)));
  load_twiddles(s_tw, LW > 0 ? a.tws : a.tw, ntw);
  if (DK == DN_CONV)
    for (int i = threadIdx.x; i < ks * ks; i += blockDim.x) s_taps[i] = a.dn.taps[i];
  const double* x0 = a0 ? a.xin.at(b0, a.st) : nullptr;
  const double* x1 = a1 ? a.xin.at(b1, a.st) : nullptr;
  const int r0 = blockIdx.x * a.lpc;
  const int trows = a.lpc + 2 * R;
  const TileLayout tl{RowLayout::stride_for(W)};
  // tile rows r0-R .. r0+lpc+R-1 (periodic), both images
  if ((W & 1) == 0) {  // even width: every row (and image) starts 16-byte aligned
    const int W2 = W >> 1;
    const int total = trows * W2;
    // batches of RF_BATCH iterations: all loads of a batch issue before its stores
    // (the tile load is the kernel's exposed latency: keep many in flight)
    for (int base = 0; base < total; base += RF_BATCH * blockDim.x) {
      double2 u0[RF_BATCH], u1[RF_BATCH];
#pragma unroll
      for (int q = 0; q < RF_BATCH; ++q) {
        const int idx = base + q * blockDim.x + threadIdx.x;
        const int i = idx / W2, c2 = idx - i * W2;
        const long long o = (long long)wrap(r0 - R + i, H) * W + 2 * c2;
        const bool in = idx < total;
        u0[q] = (in && x0) ? __ldg(reinterpret_cast<const double2*>(x0 + o)) : make_double2(0.0, 0.0);
        u1[q] = (in && x1) ? __ldg(reinterpret_cast<const double2*>(x1 + o)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < RF_BATCH; ++q) {
        const int idx = base + q * blockDim.x + threadIdx.x;
        if (idx >= total) break;
        const int i = idx / W2, c2 = idx - i * W2;
        st_cd(s_work + tl.at(i, 2 * c2), cd{u0[q].x, u1[q].x});
        st_cd(s_work + tl.at(i, 2 * c2 + 1), cd{u0[q].y, u1[q].y});
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < trows * W; idx += blockDim.x) {
      const int i = idx / W, c = idx - i * W;
      const long long o = (long long)wrap(r0 - R + i, H) * W + c;
      st_cd(s_work + tl.at(i, c), cd{x0 ? __ldg(x0 + o) : 0.0, x1 ? __ldg(x1 + o) : 0.0});
    }
  }
  __syncthreads();
  const int line = threadIdx.x / T, t = threadIdx.x - line * T;
  const int row = r0 + line;
  const bool valid = row < H;
  const int ti = line + R;  // tile row of this output row
  const int c0 = 16 * t;    // this thread's contiguous span [c0, c0+16)
  cd f[16];
  denoise_span<DK>(f, s_work, tl, ti, c0, ks, s_taps, [&](int c) { return colwrap<LW>(c, W); });
  __syncthreads();  // tile no longer read: reuse it as the line buffer
  RowLayout lay{RowLayout::stride_for(W)};
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (c0 + j < W) st_cd(s_work + lay.at(line, c0 + j), f[j]);
  __syncthreads();
  if (a.fout) {  // keep f(x) for the cost identity of this step (cadence only), coalesced
    const long long N = (long long)H * W;
    const int nl = min(a.lpc, H - r0);
    for (int idx = threadIdx.x; idx < nl * W; idx += blockDim.x) {
      const int l = idx / W, c = idx - l * W;
      const cd fv = ld_cd(s_work + lay.at(l, c));
      const long long o = (long long)(r0 + l) * W + c;
      if (a0) a.fout[(long long)b0 * N + o] = fv.x;
      if (a1) a.fout[(long long)b1 * N + o] = fv.y;
    }
  }
  cd v[16];
  if constexpr (LW > 0) {
    line_fft_ct<LW, false, true>(v, s_work, s_tw, t, line, lay);
  } else {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int c = t + T * m;
      v[m] = c < W ? ld_cd(s_work + lay.at(line, c)) : cd{0.0, 0.0};
    }
    __syncthreads();
    line_fft<false>(v, s_work, s_tw, W, t, line, lay);
  }
  if (valid) {
    cd* zr = a.Z + ((long long)p * H + row) * W;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int c = t + T * m;
      if (c < W) st_cd(zr + c, v[m]);
    }
  }
}

template <class K>
static void big_smem_once(K kernel, bool& done) {
  if (done) return;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)fa.sharedSizeBytes);
  done = true;
}

template <int LW, int DK>
static void row_fwd_t(const RowFwdArgs& a, int npairs, cudaStream_t s) {
  static bool done = false;
  big_smem_once(k_row_fwd<LW, DK>, done);
  const int T = threads_per_line(a.W);
  dim3 grid(cdivf(a.H, a.lpc), npairs);
  k_row_fwd<LW, DK><<<grid, a.lpc * T, row_fwd_smem(a.W, a.lpc, a.dn.radius, a.dn.ksize), s>>>(a);
}

template <int DK>
static void row_fwd_dk(const RowFwdArgs& a, int npairs, cudaStream_t s) {
  switch (a.W) {
    case 64: row_fwd_t<64, DK>(a, npairs, s); break;
    case 128: row_fwd_t<128, DK>(a, npairs, s); break;
    case 256: row_fwd_t<256, DK>(a, npairs, s); break;
    case 512: row_fwd_t<512, DK>(a, npairs, s); break;
    case 1024: row_fwd_t<1024, DK>(a, npairs, s); break;
    default: row_fwd_t<0, DK>(a, npairs, s); break;
  }
}

void launch_row_fwd(const RowFwdArgs& a, int npairs, cudaStream_t s) {
  switch (a.dn.kind) {
    case DN_CONV: row_fwd_dk<DN_CONV>(a, npairs, s); break;
    case DN_MEDIAN3: row_fwd_dk<DN_MEDIAN3>(a, npairs, s); break;
    default: row_fwd_dk<DN_IDENTITY>(a, npairs, s); break;
  }
}

// --------------------------------------------------------------- columns
template <int LH>
__global__ void __launch_bounds__(128, 3) k_col(ColArgs a) {
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const bool a0 = takes_step(a.st[b0], a.phase);
  const bool a1 = b1 < a.B && takes_step(a.st[b1], a.phase);
  if (!a0 && !a1) return;
  const int H = LH > 0 ? LH : a.H;
  const int W = a.W;
  const int T = LH > 0 ? LH / 16 : threads_per_line(H);
  const int ntw = LH > 0 ? tw_stage_size(LH) : H;
  cd* s_tw = reinterpret_cast<cd*>(f_smem);
  cd* s_work = reinterpret_cast<cd*>(f_smem + al16f(ntw * sizeof(cd)));
  load_twiddles(s_tw, LH > 0 ? a.tws : a.tw, ntw);
  const int line = threadIdx.x % a.lpc, t = threadIdx.x / a.lpc;
  const int col = blockIdx.x * a.lpc + line;
  const bool valid = col < W;
  cd* zc = a.Z + (long long)p * H * W + (valid ? col : 0);
  // the spectral multiplier for this thread's 16 elements: async copies into
  // shared memory now, consumed after the forward transform
  double* s_g = reinterpret_cast<double*>(s_work + (size_t)H * a.lpc);
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int r = t + T * m;
    if (valid && r < H) {
      const unsigned dst =
          (unsigned)__cvta_generic_to_shared(s_g + m * blockDim.x + threadIdx.x);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                   "l"(a.g + (long long)r * W + col));
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
  cd v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int r = t + T * m;
    v[m] = (valid && r < H) ? ld_cd(zc + (long long)r * W) : cd{0.0, 0.0};
  }
  __syncthreads();
  ColLayout lay{a.lpc};
  fft_dispatch<LH, false>(v, s_work, s_tw, H, t, line, lay);
  asm volatile("cp.async.wait_group 0;\n" ::);  // this thread's own copies
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int r = t + T * m;
    if (valid && r < H) v[m] = v[m] * (a.scale * s_g[m * blockDim.x + threadIdx.x]);
  }
  fft_dispatch<LH, true>(v, s_work, s_tw, H, t, line, lay);
  if (valid) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const int r = t + T * m;
      if (r < H) st_cd(zc + (long long)r * W, v[m]);
    }
  }
}

template <int LH>
static void col_t(const ColArgs& a, int npairs, cudaStream_t s) {
  static bool done = false;
  big_smem_once(k_col<LH>, done);
  const int T = threads_per_line(a.H);
  dim3 grid(cdivf(a.W, a.lpc), npairs);
  k_col<LH><<<grid, a.lpc * T, col_smem(a.H, a.lpc), s>>>(a);
}

void launch_col(const ColArgs& a, int npairs, cudaStream_t s) {
  switch (a.H) {
    case 64: col_t<64>(a, npairs, s); break;
    case 128: col_t<128>(a, npairs, s); break;
    case 256: col_t<256>(a, npairs, s); break;
    case 512: col_t<512>(a, npairs, s); break;
    case 1024: col_t<1024>(a, npairs, s); break;
    default: col_t<0>(a, npairs, s); break;
  }
}

// --------------------------------------------------------------- row inverse
template <int LW>
__global__ void __launch_bounds__(128, 4) k_row_inv(RowInvArgs a) {
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const int phase = a.epilogue ? a.ctl.phase : PH_SETUP;
  const bool a0 = takes_step(a.st[b0], phase);
  const bool a1 = b1 < a.B && takes_step(a.st[b1], phase);
  if (!a0 && !a1) return;
  const int W = LW > 0 ? LW : a.W;
  const int H = a.H;
  const int T = LW > 0 ? LW / 16 : threads_per_line(W);
  const long long N = (long long)H * W;
  const int ntw = LW > 0 ? tw_stage_size(LW) : W;
  cd* s_tw = reinterpret_cast<cd*>(f_smem);
  cd* s_work = reinterpret_cast<cd*>(f_smem + al16f(ntw * sizeof(cd)));
  double* s_red = reinterpret_cast<double*>(f_smem + al16f(ntw * sizeof(cd)) +
                                            (size_t)a.lpc * RowLayout::stride_for(W) * sizeof(cd));
  load_twiddles(s_tw, LW > 0 ? a.tws : a.tw, ntw);
  const int line = threadIdx.x / T, t = threadIdx.x - line * T;
  const int row = blockIdx.x * a.lpc + line;
  const bool valid = row < H;
  const cd* zr = a.Z + ((long long)p * H + (valid ? row : 0)) * W;
  cd v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int c = t + T * m;
    v[m] = (valid && c < W) ? ld_cd(zr + c) : cd{0.0, 0.0};
  }
  __syncthreads();
  RowLayout lay{RowLayout::stride_for(W)};
  fft_dispatch<LW, true>(v, s_work, s_tw, W, t, line, lay);

  double acc[6] = {0, 0, 0, 0, 0, 0};
  if (valid) {
    double* o0 = a0 ? a.out.at(b0, a.st) + (long long)row * W : nullptr;
    double* o1 = a1 ? a.out.at(b1, a.st) + (long long)row * W : nullptr;
    const double* p0 = (a0 && a.epilogue) ? a.xprev.at(b0, a.st) + (long long)row * W : nullptr;
    const double* p1 = (a1 && a.epilogue) ? a.xprev.at(b1, a.st) + (long long)row * W : nullptr;
    const double* bs0 = (a0 && a.base) ? a.base + (long long)b0 * N + (long long)row * W : nullptr;
    const double* bs1 = (a1 && a.base) ? a.base + (long long)b1 * N + (long long)row * W : nullptr;
    // four batches of 4 columns: all loads of a batch issue before its stores
    // (8-column batches spilled at the 128-register cap)
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      double lb0[4], lb1[4], lp0[4], lp1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = t + T * (4 * h + q);
        const bool in = c < W;
        lb0[q] = (in && bs0) ? __ldg(bs0 + c) : 0.0;
        lb1[q] = (in && bs1) ? __ldg(bs1 + c) : 0.0;
        lp0[q] = (in && p0) ? __ldg(p0 + c) : 0.0;
        lp1[q] = (in && p1) ? __ldg(p1 + c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int m = 4 * h + q;
        const int c = t + T * m;
        if (c >= W) continue;
        if (o0) {
          const double val = v[m].x + lb0[q];
          o0[c] = val;
          if (p0) {
            const double d = val - lp0[q];
            acc[0] = fma(d, d, acc[0]);
            acc[1] = fma(lp0[q], lp0[q], acc[1]);
            acc[2] += isfinite(val) ? 0.0 : 1.0;
          }
        }
        if (o1) {
          const double val = v[m].y + lb1[q];
          o1[c] = val;
          if (p1) {
            const double d = val - lp1[q];
            acc[3] = fma(d, d, acc[3]);
            acc[4] = fma(lp1[q], lp1[q], acc[4]);
            acc[5] += isfinite(val) ? 0.0 : 1.0;
          }
        }
      }
    }
  }
  if (!a.epilogue) return;
  block_sum<6>(acc, s_red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0) {
    double* dst = a.partials + ((long long)p * nblk + blockIdx.x) * 6;
#pragma unroll
    for (int i = 0; i < 6; ++i) dst[i] = acc[i];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + p, nblk, &s_last);
  double tot[6];
  if (lastb) gather_partials<6>(a.partials + (long long)p * nblk * 6, nblk, tot, s_red);
  if (lastb && threadIdx.x == 0) {
    if (a0) record_step(a.st[b0], b0, tot[0], tot[1], tot[2], a.S, a.ctl, a.tr);
    if (a1) record_step(a.st[b1], b1, tot[3], tot[4], tot[5], a.S, a.ctl, a.tr);
  }
}

template <int LW>
static void row_inv_t(const RowInvArgs& a, int npairs, cudaStream_t s) {
  static bool done = false;
  big_smem_once(k_row_inv<LW>, done);
  const int T = threads_per_line(a.W);
  dim3 grid(cdivf(a.H, a.lpc), npairs);
  k_row_inv<LW><<<grid, a.lpc * T, row_inv_smem(a.W, a.lpc), s>>>(a);
}

void launch_row_inv(const RowInvArgs& a, int npairs, cudaStream_t s) {
  switch (a.W) {
    case 64: row_inv_t<64>(a, npairs, s); break;
    case 128: row_inv_t<128>(a, npairs, s); break;
    case 256: row_inv_t<256>(a, npairs, s); break;
    case 512: row_inv_t<512>(a, npairs, s); break;
    case 1024: row_inv_t<1024>(a, npairs, s); break;
    default: row_inv_t<0>(a, npairs, s); break;
  }
}

}  // namespace redve
