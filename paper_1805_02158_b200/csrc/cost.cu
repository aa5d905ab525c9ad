// Fused objective evaluation, fast path: E(x) = ||Hx - y||^2/(2 sigma^2)
// + alpha/2 x.(x - f(x)) and the PSNR sum, for a rank-one PSF and widths that
// are multiples of 16 (objective.py:78-88, imaging.py:234-248).
//
// One CTA = `rows` output rows of an image pair; each thread owns 16
// contiguous columns of one row.  The blur is two 1-D passes (vertical into
// shared memory, horizontal from a register window), the denoiser is the
// shared-column median / stencil of cost.cuh; partial sums are reduced
// deterministically (per-CTA partials, last CTA of the pair sums in order).
#include "cost.cuh"
#include "kernels.cuh"

namespace redve {

extern __shared__ __align__(16) unsigned char c_smem[];

static inline __host__ __device__ size_t al16c(size_t b) { return (b + 15) & ~size_t(15); }

int cost_fast_rows(int W) {
  const int spans = W / 16;
  int rows = 128 / spans;
  return rows < 1 ? 1 : rows;
}

bool cost_fast_ok(const CostArgs& a) {
  return a.separable && (a.W % 16) == 0 && a.W >= 16 && a.hk / 2 < 16;
}

size_t cost_fast_smem(const CostArgs& a, int rows) {
  const int rH = a.hk / 2;
  const int Rd = a.dn.kind == DN_CONV ? a.dn.ksize / 2 : (a.dn.kind == DN_MEDIAN3 ? 1 : 0);
  const int R = rH > Rd ? rH : Rd;
  const int kk = a.dn.kind == DN_CONV ? a.dn.ksize * a.dn.ksize : 0;
  const int st = TileLayout::stride_for(a.W);
  return al16c((2 * a.hk + kk + 32 * 6) * sizeof(double)) +
         (size_t)(rows + 2 * R) * st * sizeof(cd) + (size_t)rows * st * sizeof(cd);
}

template <int DK>
__global__ void __launch_bounds__(256) k_cost_fast(CostArgs a) {
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const bool has1 = b1 < a.B;
  const bool w0 = cost_wants(a.st[b0], a);
  const bool w1 = has1 && cost_wants(a.st[b1], a);
  const int nblk = gridDim.x;
  if (!w0 && !w1) {
    if (a.mode == COST_RECORD && blockIdx.x == 0 && threadIdx.x == 0) {
      commit_step(a.st[b0], a.ctl.phase);
      if (has1) commit_step(a.st[b1], a.ctl.phase);
    }
    return;
  }
  const int W = a.W, H = a.H, rows = a.rows;
  const long long N = (long long)H * W;
  const int rH = a.hk / 2;
  const int Rd = DK == DN_CONV ? a.dn.ksize / 2 : (DK == DN_MEDIAN3 ? 1 : 0);
  const int R = rH > Rd ? rH : Rd;
  const int kk = DK == DN_CONV ? a.dn.ksize * a.dn.ksize : 0;
  const TileLayout tl{TileLayout::stride_for(W)};
  double* s_u = reinterpret_cast<double*>(c_smem);
  double* s_v = s_u + a.hk;
  double* s_taps = s_v + a.hk;
  double* s_red = s_taps + kk;
  cd* tile = reinterpret_cast<cd*>(c_smem + al16c((2 * a.hk + kk + 32 * 6) * sizeof(double)));
  cd* vbuf = tile + (size_t)(rows + 2 * R) * tl.stride;
  for (int i = threadIdx.x; i < a.hk; i += blockDim.x) {
    s_u[i] = a.hu[i];
    s_v[i] = a.hv[i];
  }
  for (int i = threadIdx.x; i < kk; i += blockDim.x) s_taps[i] = a.dn.taps[i];
  const double* x0 = w0 ? a.x.at(b0, a.st) : nullptr;
  const double* x1 = w1 ? a.x.at(b1, a.st) : nullptr;
  const int r0 = blockIdx.x * rows;
  const int trows = rows + 2 * R;
  {  // tile rows r0-R .. r0+rows+R-1, both images (W even: 16-byte loads)
    const int W2 = W >> 1;
    const int total = trows * W2;
    for (int base = 0; base < total; base += 4 * blockDim.x) {
      double2 u0[4], u1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = base + q * blockDim.x + threadIdx.x;
        const int i = idx / W2, c2 = idx - i * W2;
        const long long o = (long long)wrap(r0 - R + i, H) * W + 2 * c2;
        const bool in = idx < total;
        u0[q] = (in && x0) ? __ldg(reinterpret_cast<const double2*>(x0 + o)) : make_double2(0.0, 0.0);
        u1[q] = (in && x1) ? __ldg(reinterpret_cast<const double2*>(x1 + o)) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int idx = base + q * blockDim.x + threadIdx.x;
        if (idx >= total) break;
        const int i = idx / W2, c2 = idx - i * W2;
        st_cd(tile + tl.at(i, 2 * c2), cd{u0[q].x, u1[q].x});
        st_cd(tile + tl.at(i, 2 * c2 + 1), cd{u0[q].y, u1[q].y});
      }
    }
  }
  __syncthreads();
  const int spans = W / 16;
  const int li = threadIdx.x / spans, t = threadIdx.x - li * spans;
  const int row = r0 + li;
  const bool valid = li < rows && row < H;
  const int c0 = 16 * t;
  const int s = a.factor;
  const bool grid_row = valid && (row % s) == 0;
  if (grid_row) {  // vertical blur pass on measurement-grid rows
#pragma unroll 4
    for (int j = 0; j < 16; ++j) {
      cd acc = cd{0.0, 0.0};
      for (int ta = 0; ta < a.hk; ++ta) {
        const cd xx = ld_cd(tile + tl.at(li + R - (ta - rH), c0 + j));
        acc.x = fma(s_u[ta], xx.x, acc.x);
        acc.y = fma(s_u[ta], xx.y, acc.y);
      }
      st_cd(vbuf + tl.at(li, c0 + j), acc);
    }
  }
  __syncthreads();
  double acc[6] = {0, 0, 0, 0, 0, 0};  // fid0, reg0, ssd0, fid1, reg1, ssd1
  if (valid) {
    const long long ro = (long long)row * W;
    cd f[16];
    if (DK == DN_EXTERNAL) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        f[j] = cd{x0 ? __ldg(a.fext + (long long)b0 * N + ro + c0 + j) : 0.0,
                  x1 ? __ldg(a.fext + (long long)b1 * N + ro + c0 + j) : 0.0};
    } else {
      denoise_span<DK>(f, tile, tl, li + R, c0, a.dn.ksize, s_taps,
                       [&](int c) { return edge_wrap(c, W); });
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const cd xv = ld_cd(tile + tl.at(li + R, c0 + j));
      acc[1] = fma(xv.x, xv.x - f[j].x, acc[1]);
      acc[4] = fma(xv.y, xv.y - f[j].y, acc[4]);
      if (a.ref) {
        if (x0) {
          const double d = xv.x - __ldg(a.ref + (long long)b0 * N + ro + c0 + j);
          acc[2] = fma(d, d, acc[2]);
        }
        if (x1) {
          const double d = xv.y - __ldg(a.ref + (long long)b1 * N + ro + c0 + j);
          acc[5] = fma(d, d, acc[5]);
        }
      }
    }
    if (grid_row) {  // horizontal pass + residual at the measurement-grid columns
      const long long Ny = (long long)a.Hy * a.Wy;
      const long long oy = (long long)(row / s) * a.Wy;
      for (int j = 0; j < 16; ++j) {
        const int c = c0 + j;
        if (c % s) continue;
        cd hx = cd{0.0, 0.0};
        for (int tb = 0; tb < a.hk; ++tb) {
          const cd vv = ld_cd(vbuf + tl.at(li, edge_wrap(c - (tb - rH), W)));
          hx.x = fma(s_v[tb], vv.x, hx.x);
          hx.y = fma(s_v[tb], vv.y, hx.y);
        }
        if (x0) {
          const double d = hx.x - __ldg(a.y + (long long)b0 * Ny + oy + c / s);
          acc[0] = fma(d, d, acc[0]);
        }
        if (x1) {
          const double d = hx.y - __ldg(a.y + (long long)b1 * Ny + oy + c / s);
          acc[3] = fma(d, d, acc[3]);
        }
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

template <int DK>
static void cost_fast_t(const CostArgs& a0, int npairs, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k_cost_fast<DK>) == cudaSuccess)
      cudaFuncSetAttribute(k_cost_fast<DK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           optin - (int)fa.sharedSizeBytes);
    done = true;
  }
  CostArgs a = a0;
  a.rows = cost_fast_rows(a.W);
  const int threads = a.rows * (a.W / 16);
  dim3 grid((a.H + a.rows - 1) / a.rows, npairs);
  k_cost_fast<DK><<<grid, threads, cost_fast_smem(a, a.rows), s>>>(a);
}

void launch_cost_fast(const CostArgs& a, int npairs, cudaStream_t s) {
  switch (a.dn.kind) {
    case DN_CONV: cost_fast_t<DN_CONV>(a, npairs, s); break;
    case DN_MEDIAN3: cost_fast_t<DN_MEDIAN3>(a, npairs, s); break;
    case DN_EXTERNAL: cost_fast_t<DN_EXTERNAL>(a, npairs, s); break;
    default: cost_fast_t<DN_IDENTITY>(a, npairs, s); break;
  }
}

// ---------------------------------------------------------------------------
// Fourier-route objective by the normal-equation identity.  x = x_k is the
// exact solution of (H^T H / s^2 + a I) x = H^T y / s^2 + a f, f = f(x_{k-1})
// (objective.py:100-104), so H^T H x = H^T y + a s^2 (f - x) and
//   ||Hx - y||^2 = ||y||^2 - s^2 <x, H^T y / s^2> + a s^2 <x, f - x>
// -- no blur of x.  A streaming pass: each thread owns a pair of adjacent
// pixels of one image, forms f(x_k) from L1-resident neighbours (median /
// stencil) or reads it (precomputed denoisers), and reads f(x_{k-1}) (kept by
// k_row_fwd), H^T y / s^2 and the reference with coalesced 16-byte loads.
int cost_fp_rows(int W) {  // kept for the partials sizing of the problem
  int rows = 2048 / W;
  return rows < 1 ? 1 : rows;
}

bool cost_fp_ok(const CostArgs& a) {
  return a.fprev && a.hty && a.yy && (a.W % 2) == 0 && a.W >= 4 && a.H >= 3 && a.factor == 1 &&
         (a.dn.kind != DN_CONV || a.dn.ksize <= 7);
}

static int cost_fp_chunks(int B, long long N, int wave) {
  // one wave at the kernel's residency (4 CTAs/SM x 148 SMs at 64 registers):
  // 1216 CTAs for B = 64 left a 3rd wave of 32 CTAs (47 us); 576 CTAs: 44 us
  int c = wave / B;
  const long long per = (N / 2 + 255) / 256;  // CTA-passes per image
  if (c > per) c = (int)per;
  if (c > 64) c = 64;
  return c < 1 ? 1 : c;
}

template <int DK>
__global__ void __launch_bounds__(256) k_cost_fp(CostArgs a) {
  const int b = blockIdx.y;
  ImgState& st = a.st[b];
  const bool want = cost_wants(st, a);
  const int nblk = gridDim.x;
  if (!want) {
    if (a.mode == COST_RECORD && blockIdx.x == 0 && threadIdx.x == 0) commit_step(st, a.ctl.phase);
    return;
  }
  __shared__ double s_taps[64];
  __shared__ double s_red[32 * 4];
  const int kk = DK == DN_CONV ? a.dn.ksize * a.dn.ksize : 0;
  for (int i = threadIdx.x; i < kk && i < 64; i += blockDim.x) s_taps[i] = a.dn.taps[i];
  if (DK == DN_CONV) __syncthreads();
  const int H = a.H, W = a.W;
  const long long N = (long long)H * W;
  const double* x = a.x.at(b, a.st);
  const double* fx = DK == DN_EXTERNAL ? a.fext + (long long)b * N : x;
  const double* hp = a.hty + (long long)b * N;
  const double* fp = a.fprev + (long long)b * N;
  const double* rp = a.ref ? a.ref + (long long)b * N : nullptr;
  const int W2 = W >> 1;
  const long long P = N >> 1;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};  // reg, <x,hty>, <x,fprev-x>, ssd
  // grid-stride over pixel pairs with the (row, pair) position advanced
  // incrementally (no division in the loop)
  const long long q0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)nblk * blockDim.x;
  const int di = (int)(stride / W2), dj = (int)(stride % W2);
  int i = (int)(q0 / W2), j2 = (int)(q0 % W2);
  for (long long q = q0; q < P; q += stride) {
    const int j = 2 * j2;
    const long long o = (long long)i * W + j;
    const double2 xv = __ldg(reinterpret_cast<const double2*>(x + o));
    const double2 hv = __ldg(reinterpret_cast<const double2*>(hp + o));
    const double2 fv = __ldg(reinterpret_cast<const double2*>(fp + o));
    double f0, f1;
    fk_pair<DK>(fx, H, W, i, j, a.dn, s_taps, f0, f1);
    acc[0] = fma(xv.x, xv.x - f0, acc[0]);
    acc[0] = fma(xv.y, xv.y - f1, acc[0]);
    acc[1] = fma(xv.x, hv.x, acc[1]);
    acc[1] = fma(xv.y, hv.y, acc[1]);
    acc[2] = fma(xv.x, fv.x - xv.x, acc[2]);
    acc[2] = fma(xv.y, fv.y - xv.y, acc[2]);
    if (rp) {
      const double2 rv = __ldg(reinterpret_cast<const double2*>(rp + o));
      const double d0 = xv.x - rv.x, d1 = xv.y - rv.y;
      acc[3] = fma(d0, d0, acc[3]);
      acc[3] = fma(d1, d1, acc[3]);
    }
    i += di;
    j2 += dj;
    if (j2 >= W2) {
      j2 -= W2;
      ++i;
    }
  }
  block_sum<4>(acc, s_red);
  if (threadIdx.x == 0) {
    double* dst = a.partials + ((long long)b * nblk + blockIdx.x) * 4;
    for (int i = 0; i < 4; ++i) dst[i] = acc[i];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double T[4];
  if (lastb) gather_partials<4>(a.partials + (long long)b * nblk * 4, nblk, T, s_red);
  if (lastb && threadIdx.x == 0) {
    const double s2 = a.sigma * a.sigma;
    const double fid = a.yy[b] + s2 * (a.alpha * T[2] - T[1]);
    if (a.mode == COST_VALUE) {
      a.out_vals[b * 3 + 0] = fid;
      a.out_vals[b * 3 + 1] = T[0];
      a.out_vals[b * 3 + 2] = T[3];
    } else {
      cost_finish(st, b, fid, T[0], T[3], a.ref != nullptr, a);
    }
    if (a.mode == COST_RECORD) commit_step(st, a.ctl.phase);
  }
}

template <int DK>
static void cost_fp_t(const CostArgs& a, cudaStream_t s) {
  // resident CTAs of this instantiation on this device, queried once
  static int wave = 0;
  if (wave == 0) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cost_fp<DK>, 256, 0);
    wave = sms * (per_sm > 0 ? per_sm : 1);
  }
  dim3 grid(cost_fp_chunks(a.B, (long long)a.H * a.W, wave), a.B);
  k_cost_fp<DK><<<grid, 256, 0, s>>>(a);
}

void launch_cost_fp(const CostArgs& a, int npairs, cudaStream_t s) {
  (void)npairs;
  switch (a.dn.kind) {
    case DN_CONV: cost_fp_t<DN_CONV>(a, s); break;
    case DN_MEDIAN3: cost_fp_t<DN_MEDIAN3>(a, s); break;
    case DN_EXTERNAL: cost_fp_t<DN_EXTERNAL>(a, s); break;
    default: cost_fp_t<DN_IDENTITY>(a, s); break;
  }
}

}  // namespace redve
