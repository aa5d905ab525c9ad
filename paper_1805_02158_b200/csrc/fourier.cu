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
#include <cudaTypedefs.h>

#include "cost.cuh"
#include "kernels.cuh"
#include "tma.cuh"

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
  const int ntw = LW > 0 ? tw_stage_size(LW) : a.W;
  // twiddle loads first: they do not depend on the image state, so they overlap
  // the tile's (state -> slot -> address) latency chain; parked after the tile
  const TwiddleRegs twq = twiddles_issue(LW > 0 ? a.tws : a.tw, ntw);
  const bool a0 = takes_step(a.st[b0], a.phase);
  const bool a1 = b1 < a.B && takes_step(a.st[b1], a.phase);
  if (!a0 && !a1) return;
  const int W = LW > 0 ? LW : a.W;
  const int H = a.H;
  const int T = LW > 0 ? LW / 16 : threads_per_line(W);
  const int R = DK == DN_CONV ? a.dn.ksize / 2 : (DK == DN_MEDIAN3 ? 1 : 0);
  const int ks = DK == DN_CONV ? a.dn.ksize : 0;
  cd* s_tw = reinterpret_cast<cd*>(f_smem);
  double* s_taps = reinterpret_cast<double*>(f_smem + al16f(ntw * sizeof(cd)));
  cd* s_work = reinterpret_cast<cd*>(f_smem + al16f(ntw * sizeof(cd)) +
                                     al16f((size_t)a.dn.ksize * a.dn.ksize * sizeof(double)));
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
  twiddles_park(s_tw, LW > 0 ? a.tws : a.tw, ntw, twq);
  if (DK == DN_CONV)
    for (int i = threadIdx.x; i < ks * ks; i += blockDim.x) s_taps[i] = a.dn.taps[i];
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
    if (valid && r < H) {  // explicit roundings: no contraction into the next butterfly
      const double gs = __dmul_rn(a.scale, s_g[m * blockDim.x + threadIdx.x]);
      v[m] = cd{__dmul_rn(v[m].x, gs), __dmul_rn(v[m].y, gs)};
    }
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

// --------------------------------------------------------------- persistent column pass
// k_col_p: one CTA per resident slot (3 per SM) walks the pass's tiles (round
// robin, tiles of inactive pairs skipped) through a ring of 2 shared-memory
// stages that TMA fills ahead of the math, so every SM keeps tiles of HBM reads
// in flight while it transforms the current one (the one-shot k_col loads a
// tile into registers, transforms, stores: its CTAs run in phase and HBM idles
// during the transforms).  Measured: 23.4 -> 23.0 us at 64 x 256^2, 209 -> 182
// us at 128 x 512^2.  The same design for the inverse row pass (x_b / x_prev /
// spectrum rows by bulk copies, producer warp + 4 math warps, 96 KB stages)
// ran 36 -> 51 us: one CTA per SM leaves too few warps to hide the FFT's own
// latencies (ncu: 7.5% warps active, consumers waiting on the stage).

bool encode_tmap_f64_3d(CUtensorMap* map, const void* base, const uint64_t dims[3],
                        const uint64_t strides_bytes[2], const uint32_t box[3]) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    cudaGetLastError();
  }
  if (!fn) return false;
  cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  cuuint64_t st[2] = {strides_bytes[0], strides_bytes[1]};
  cuuint32_t bx[3] = {box[0], box[1], box[2]};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), d, st, bx, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class K>
static int resident_ctas(K kernel, int threads, size_t smem) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  return sms * (per > 0 ? per : 1);
}

constexpr int P_MAX_IMAGES = 4096;  // per-image step flags in shared memory

// Which images take this step, built once per CTA with one round of parallel
// state loads (the tile loop then never waits on global memory to decide).
__device__ __forceinline__ void step_flags(unsigned char* f, const ImgState* st, int B, int phase) {
  for (int b = threadIdx.x; b < B; b += blockDim.x) f[b] = takes_step(st[b], phase) ? 1 : 0;
}
__device__ __forceinline__ bool pair_on(const unsigned char* f, int B, int p) {
  return f[2 * p] || (2 * p + 1 < B && f[2 * p + 1]);
}

constexpr int CP_NS = 2;  // column pass: 2 stages of 32 KB, 3 CTAs per SM

template <int LH>
constexpr size_t col_p_smem() {
  return al16f(tw_stage_size(LH) * sizeof(cd)) + (size_t)CP_NS * 128 * 16 * sizeof(cd) +
         CP_NS * sizeof(uint64_t) + P_MAX_IMAGES;
}

// Column pass, persistent: tile = LPC whole columns of one pair (LH x LPC
// complex, 32 KB), landed by 3-D TMA boxes in the column layout the FFT reads
// (element r of column c at r*LPC + c), transformed in place, scaled by alpha g
// (L2-resident, per column block), inverse transformed, stored coalesced.
template <int LH>
__global__ void __launch_bounds__(128, 3) k_col_p(const __grid_constant__ CUtensorMap tm, ColArgs a,
                                                  int npairs) {
  constexpr int T = LH / 16, LPC = 128 / T, TILE = LH * LPC;
  constexpr int BOXR = LH < 256 ? LH : 256;
  cd* s_tw = reinterpret_cast<cd*>(f_smem);
  cd* s_st = reinterpret_cast<cd*>(f_smem + al16f(tw_stage_size(LH) * sizeof(cd)));
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(s_st + CP_NS * TILE);
  unsigned char* s_img = reinterpret_cast<unsigned char*>(s_bar + CP_NS);
  const int W = a.W, ncb = W / LPC, ntiles = npairs * ncb, G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CP_NS; ++s) mbar_init(&s_bar[s], 1);
    fence_mbar_init();
  }
  step_flags(s_img, a.st, a.B, a.phase);
  load_twiddles(s_tw, a.tws, tw_stage_size(LH));
  __syncthreads();
  auto next = [&](int i) {
    while (i < ntiles && !pair_on(s_img, a.B, i / ncb)) i += G;
    return i;
  };
  auto issue = [&](int s, int i) {
    const int p = i / ncb, cb = i - p * ncb;
    mbar_arrive_expect_tx(&s_bar[s], TILE * (uint32_t)sizeof(cd));
#pragma unroll
    for (int rb = 0; rb < LH; rb += BOXR)
      tma_load_3d(s_st + s * TILE + rb * LPC, &tm, cb * 2 * LPC, rb, p, &s_bar[s]);
  };
  int fill = 0;
  if (threadIdx.x == 0) {
    fill = next(blockIdx.x);
    for (int s = 0; s < CP_NS && fill < ntiles; ++s) {
      issue(s, fill);
      fill = next(fill + G);
    }
  }
  const int line = threadIdx.x % LPC, t = threadIdx.x / LPC;
  const ColLayout lay{LPC};
  int k = 0;
  for (int cur = next(blockIdx.x); cur < ntiles; cur = next(cur + G), ++k) {
    const int s = k % CP_NS;
    const int p = cur / ncb, col = (cur - p * ncb) * LPC + line;
    double gv[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) gv[m] = __ldg(a.g + (long long)(t + T * m) * W + col);
    mbar_wait(&s_bar[s], (uint32_t)(k / CP_NS) & 1u);
    cd* buf = s_st + s * TILE;
    cd v[16];
    line_fft_ct<LH, false, true>(v, buf, s_tw, t, line, lay);
#pragma unroll
    for (int m = 0; m < 16; ++m) {  // rounded as k_col (no contraction)
      const double gs = __dmul_rn(a.scale, gv[m]);
      v[m] = cd{__dmul_rn(v[m].x, gs), __dmul_rn(v[m].y, gs)};
    }
    line_fft_ct<LH, true>(v, buf, s_tw, t, line, lay);
    // the inverse transform's last stage ended on a barrier after its reads:
    // the stage is free for the tile CP_NS ahead
    if (threadIdx.x == 0 && fill < ntiles) {
      fence_proxy_async_smem();
      issue(s, fill);
      fill = next(fill + G);
    }
    cd* zc = a.Z + (long long)p * LH * W + col;
#pragma unroll
    for (int m = 0; m < 16; ++m) st_cd(zc + (long long)(t + T * m) * W, v[m]);
  }
}

template <int LH>
static bool col_p_t(const ColArgs& a, int npairs, cudaStream_t s) {
  constexpr int T = LH / 16, LPC = 128 / T;
  if (a.H != LH || a.W % LPC != 0 || !a.tws || a.B > P_MAX_IMAGES) return false;
  CUtensorMap tm;
  const uint64_t dims[3] = {(uint64_t)2 * a.W, (uint64_t)LH, (uint64_t)npairs};
  const uint64_t strides[2] = {(uint64_t)2 * a.W * sizeof(double),
                               (uint64_t)2 * a.W * LH * sizeof(double)};
  const uint32_t box[3] = {(uint32_t)(2 * LPC), (uint32_t)(LH < 256 ? LH : 256), 1u};
  if (!encode_tmap_f64_3d(&tm, a.Z, dims, strides, box)) return false;
  static int grid_max = 0;
  if (grid_max == 0) {
    cudaFuncSetAttribute(k_col_p<LH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)col_p_smem<LH>());
    grid_max = resident_ctas(k_col_p<LH>, 128, col_p_smem<LH>());
  }
  const int ntiles = npairs * (a.W / LPC);
  k_col_p<LH><<<ntiles < grid_max ? ntiles : grid_max, 128, col_p_smem<LH>(), s>>>(tm, a, npairs);
  return true;
}

// REDVE_PERSISTENT=0: the one-shot column kernel (A/B tests; read per launch,
// so a problem's graph keeps what its capture saw)
static bool persistent_enabled() {
  const char* e = getenv("REDVE_PERSISTENT");
  return !(e && e[0] == '0');
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
  if (persistent_enabled()) {
    bool done = false;
    switch (a.H) {
      case 128: done = col_p_t<128>(a, npairs, s); break;
      case 256: done = col_p_t<256>(a, npairs, s); break;
      case 512: done = col_p_t<512>(a, npairs, s); break;
      default: break;
    }
    if (done) return;
  }
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
// Epilogue of one image of the pair: x+ = IDFT part + x_b, and the step-norm
// partials against x_prev (acc[0..2]); all loads issue before the first use.
template <class F>
__device__ __forceinline__ void row_inv_image(double* __restrict__ o, const double* __restrict__ bs,
                                              const double* __restrict__ pv, int t, int T,
                                              double* acc, F val_of) {
  double lb[16], lp[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) lb[m] = bs ? __ldg(bs + t + T * m) : 0.0;
  if (pv) {
#pragma unroll
    for (int m = 0; m < 16; ++m) lp[m] = __ldg(pv + t + T * m);
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const double val = val_of(m) + lb[m];
    o[t + T * m] = val;
    if (pv) {
      const double d = val - lp[m];
      acc[0] = fma(d, d, acc[0]);
      acc[1] = fma(lp[m], lp[m], acc[1]);
      acc[2] += isfinite(val) ? 0.0 : 1.0;
    }
  }
}

template <int LW>
__global__ void __launch_bounds__(128, 4) k_row_inv(RowInvArgs a) {
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const int W = LW > 0 ? LW : a.W;
  const int H = a.H;
  const int T = LW > 0 ? LW / 16 : threads_per_line(W);
  const long long N = (long long)H * W;
  const int line = threadIdx.x / T, t = threadIdx.x - line * T;
  const int row = blockIdx.x * a.lpc + line;
  const bool valid = row < H;
  // the spectrum rows first: their address does not depend on the image state,
  // so the loads are in flight while the state (a dependent L2 round trip) and
  // the twiddles arrive
  const cd* zr = a.Z + ((long long)p * H + (valid ? row : 0)) * W;
  cd v[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int c = t + T * m;
    v[m] = (valid && c < W) ? ld_cd(zr + c) : cd{0.0, 0.0};
  }
  const int ntw = LW > 0 ? tw_stage_size(LW) : W;
  const TwiddleRegs twq = twiddles_issue(LW > 0 ? a.tws : a.tw, ntw);
  const int phase = a.epilogue ? a.ctl.phase : PH_SETUP;
  const bool a0 = takes_step(a.st[b0], phase);
  const bool a1 = b1 < a.B && takes_step(a.st[b1], phase);
  if (!a0 && !a1) return;
  cd* s_tw = reinterpret_cast<cd*>(f_smem);
  cd* s_work = reinterpret_cast<cd*>(f_smem + al16f(ntw * sizeof(cd)));
  double* s_red = reinterpret_cast<double*>(f_smem + al16f(ntw * sizeof(cd)) +
                                            (size_t)a.lpc * RowLayout::stride_for(W) * sizeof(cd));
  twiddles_park(s_tw, LW > 0 ? a.tws : a.tw, ntw, twq);
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
    if constexpr (LW > 0) {
      // One image at a time, all 16 columns: 32 loads in flight per thread and
      // two memory round trips per CTA instead of four (the epilogue's latency
      // is the kernel's critical path).  The second image's values wait in the
      // line buffer, which the transform's last barrier left free; each thread
      // parks and re-reads its own slots (conflict-free, no barrier).
      double* park = reinterpret_cast<double*>(s_work) + threadIdx.x;
      const int PS = blockDim.x;
      if (o1) {
#pragma unroll
        for (int m = 0; m < 16; ++m) park[m * PS] = v[m].y;
      }
      if (o0) row_inv_image(o0, bs0, p0, t, T, acc, [&](int m) { return v[m].x; });
      if (o1) row_inv_image(o1, bs1, p1, t, T, acc + 3, [&](int m) { return park[m * PS]; });
    } else {
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
