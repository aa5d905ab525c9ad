// One-kernel Fourier fixed-point step for 256 x 256 images (configs[0]/[1]):
//
//   x+ = x_b + IDFT( alpha g . DFT f(x) )              (objective.py:100-104)
//
// the same algebra and pair packing as fourier.cu's three kernels, but the
// spectrum never leaves the SMs.  A thread-block cluster of 8 CTAs owns one
// image pair; CTA r holds rows [32r, 32r+32) of the pair in shared memory:
//
//   1. x rows (+ denoiser halo) -> f(x) -> row FFTs, in place
//   2. columns [32r, 32r+32) gathered from the 8 CTAs over DSMEM, column FFT,
//      x alpha g, inverse column FFT, scattered back over DSMEM
//   3. inverse row FFTs -> + x_b -> x+, step-norm partials, last-CTA record
//
// HBM sees x (+halo), x_b, x_prev read and x+ written once per step; the
// 2 x 128 KB per CTA transpose rides DSMEM.  Register contract and FFT plans
// are fft.cuh's (compile-time L = 256, radix 16).
#include <cooperative_groups.h>

#include "cost.cuh"
#include "fused.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace redve {

extern __shared__ __align__(16) unsigned char fu_smem[];

constexpr int FU_L = 256;               // image edge
constexpr int FU_CL = 8;                // CTAs per cluster (one image pair)
constexpr int FU_ROWS = FU_L / FU_CL;   // rows (and columns) per CTA
constexpr int FU_T = FU_L / 16;         // threads per line
constexpr int FU_THREADS = FU_ROWS * FU_T;

static inline __host__ __device__ size_t al16u(size_t b) { return (b + 15) & ~size_t(15); }

static int fu_radius(const DenoiseArgs& d) {
  return d.kind == DN_CONV ? d.ksize / 2 : (d.kind == DN_MEDIAN3 ? 1 : 0);
}

static size_t fused_smem(const DenoiseArgs& d) {
  const int st = RowLayout::stride_for(FU_L);
  size_t zl = (size_t)(FU_ROWS + 2 * fu_radius(d)) * st * sizeof(cd);
  const size_t colscratch = (size_t)FU_L * FU_ROWS * sizeof(cd);
  if (colscratch > zl) zl = colscratch;
  const int kk = d.kind == DN_CONV ? d.ksize * d.ksize : 0;
  return al16u(tw_stage_size(FU_L) * sizeof(cd)) + al16u(kk * sizeof(double)) +
         al16u(32 * 6 * sizeof(double)) + zl;
}

bool fused_step_ok(int H, int W, const DenoiseArgs& d) {
  if (H != FU_L || W != FU_L) return false;
  if (d.kind != DN_MEDIAN3 && d.kind != DN_CONV && d.kind != DN_IDENTITY) return false;
  if (d.kind == DN_CONV && d.ksize > 9) return false;
  // opt-in (REDVE_FUSED=1): measured slower than the three-kernel pipeline on
  // configs[1] (148 vs 92 us per step: one 16-warp CTA per SM, 2.1 cluster
  // waves, serial phases) -- kept as a verified alternative, see DESIGN.md
  const char* e = getenv("REDVE_FUSED");
  if (!(e && e[0] == '1')) return false;
  return fused_smem(d) <= 200 * 1024;
}

template <int DK>
__global__ void __cluster_dims__(FU_CL, 1, 1) __launch_bounds__(FU_THREADS, 1)
    k_fused_step(FusedArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int p = blockIdx.y, b0 = 2 * p, b1 = 2 * p + 1;
  const int phase = a.ctl.phase;
  const bool a0 = takes_step(a.st[b0], phase);
  const bool a1 = b1 < a.B && takes_step(a.st[b1], phase);
  if (!a0 && !a1) return;  // same decision in every CTA of the cluster
  constexpr int W = FU_L, H = FU_L;
  constexpr long long N = (long long)H * W;
  const int R = DK == DN_CONV ? a.dn.ksize / 2 : (DK == DN_MEDIAN3 ? 1 : 0);
  const int ks = DK == DN_CONV ? a.dn.ksize : 0;
  constexpr int ntw = tw_stage_size(FU_L);
  cd* s_tw = reinterpret_cast<cd*>(fu_smem);
  double* s_taps = reinterpret_cast<double*>(fu_smem + al16u(ntw * sizeof(cd)));
  double* s_red = reinterpret_cast<double*>(fu_smem + al16u(ntw * sizeof(cd)) +
                                            al16u((size_t)ks * ks * sizeof(double)));
  cd* zl = reinterpret_cast<cd*>(reinterpret_cast<unsigned char*>(s_red) +
                                 al16u(32 * 6 * sizeof(double)));
  if (threadIdx.x < 4) {  // x_b / x_prev rows of this CTA (phase 3) on their way into L2
    const int bi = (threadIdx.x & 1) ? b1 : b0;
    const bool act = (threadIdx.x & 1) ? a1 : a0;
    const double* src = act ? ((threadIdx.x < 2) ? a.base + (long long)bi * N : a.xprev.at(bi, a.st))
                            : nullptr;
    if (src)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (long long)blockIdx.x * FU_ROWS * W),
                   "r"((unsigned)(FU_ROWS * W * sizeof(double))) : "memory");
  }
  load_twiddles(s_tw, a.tws, ntw);
  if (DK == DN_CONV)
    for (int i = threadIdx.x; i < ks * ks; i += blockDim.x) s_taps[i] = a.dn.taps[i];
  const double* x0 = a0 ? a.xin.at(b0, a.st) : nullptr;
  const double* x1 = a1 ? a.xin.at(b1, a.st) : nullptr;
  const int r0 = rank * FU_ROWS;
  const int tid = threadIdx.x;
  const TileLayout tl{RowLayout::stride_for(W)};
  const RowLayout lay{RowLayout::stride_for(W)};

  // ---- 1. tile rows r0-R .. r0+31+R of both images (16-byte loads, all in flight)
  {
    constexpr int W2 = W / 2;
    const int total = (FU_ROWS + 2 * R) * W2;
    constexpr int NB = 10;  // 36 rows x 128 / 512 threads <= 9
    double2 u0[NB], u1[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int idx = q * FU_THREADS + tid;
      const int i = idx / W2, c2 = idx - i * W2;
      const long long o = (long long)wrap_fast(r0 - R + i, H) * W + 2 * c2;
      const bool in = idx < total;
      u0[q] = (in && x0) ? __ldg(reinterpret_cast<const double2*>(x0 + o)) : make_double2(0.0, 0.0);
      u1[q] = (in && x1) ? __ldg(reinterpret_cast<const double2*>(x1 + o)) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const int idx = q * FU_THREADS + tid;
      if (idx >= total) break;
      const int i = idx / W2, c2 = idx - i * W2;
      st_cd(zl + tl.at(i, 2 * c2), cd{u0[q].x, u1[q].x});
      st_cd(zl + tl.at(i, 2 * c2 + 1), cd{u0[q].y, u1[q].y});
    }
  }
  __syncthreads();
  const int li = tid / FU_T, t = tid - li * FU_T;  // row line, thread in line
  {
    cd f[16];
    denoise_span<DK>(f, zl, tl, li + R, 16 * t, ks, s_taps, [&](int c) { return edge_wrap(c, W); });
    __syncthreads();  // tile consumed: the same rows become the line buffer
#pragma unroll
    for (int j = 0; j < 16; ++j) st_cd(zl + lay.at(li, 16 * t + j), f[j]);
  }
  __syncthreads();
  if (a.fout) {  // f(x) for the cost identity of this step (cadence only)
    for (int idx = tid; idx < FU_ROWS * W; idx += FU_THREADS) {
      const int l = idx / W, c = idx - l * W;
      const cd fv = ld_cd(zl + lay.at(l, c));
      const long long o = (long long)(r0 + l) * W + c;
      if (a0) a.fout[(long long)b0 * N + o] = fv.x;
      if (a1) a.fout[(long long)b1 * N + o] = fv.y;
    }
  }
  cd v[16];
  line_fft_ct<FU_L, false, true>(v, zl, s_tw, t, li, lay);
#pragma unroll
  for (int m = 0; m < 16; ++m) st_cd(zl + lay.at(li, t + FU_T * m), v[m]);
  cluster.sync();  // every CTA's row spectra complete and visible

  // ---- 2. columns [r0, r0+32): gather over DSMEM, FFT, x alpha g, inverse FFT
  const int cl = tid & (FU_ROWS - 1), tc = tid / FU_ROWS;  // column line, thread in column
  const int col = r0 + cl;
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int row = tc + FU_T * m;
    const cd* rz = cluster.map_shared_rank(zl, row / FU_ROWS);
    v[m] = ld_cd(rz + lay.at(row % FU_ROWS, col));
  }
  cluster.sync();  // all gathers done: the line buffers become column scratch
  const ColLayout clay{FU_ROWS};
  line_fft_ct<FU_L, false, false>(v, zl, s_tw, tc, cl, clay);
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int row = tc + FU_T * m;
    v[m] = v[m] * (a.scale * __ldg(a.g + (long long)row * W + col));
  }
  line_fft_ct<FU_L, true, false>(v, zl, s_tw, tc, cl, clay);
  cluster.sync();  // all column scratch use done
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int row = tc + FU_T * m;
    cd* rz = cluster.map_shared_rank(zl, row / FU_ROWS);
    st_cd(rz + lay.at(row % FU_ROWS, col), v[m]);
  }
  cluster.sync();  // rows complete again

  // ---- 3. inverse row FFTs, + x_b, x+ and the step-norm partials
  line_fft_ct<FU_L, true, true>(v, zl, s_tw, t, li, lay);
  const int row = r0 + li;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  {
    double* o0 = a0 ? a.out.at(b0, a.st) + (long long)row * W : nullptr;
    double* o1 = a1 ? a.out.at(b1, a.st) + (long long)row * W : nullptr;
    const double* p0 = a0 ? a.xprev.at(b0, a.st) + (long long)row * W : nullptr;
    const double* p1 = a1 ? a.xprev.at(b1, a.st) + (long long)row * W : nullptr;
    const double* bs0 = a0 ? a.base + (long long)b0 * N + (long long)row * W : nullptr;
    const double* bs1 = a1 ? a.base + (long long)b1 * N + (long long)row * W : nullptr;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      double lb0[4], lb1[4], lp0[4], lp1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = t + FU_T * (4 * h + q);
        lb0[q] = bs0 ? __ldg(bs0 + c) : 0.0;
        lb1[q] = bs1 ? __ldg(bs1 + c) : 0.0;
        lp0[q] = p0 ? __ldg(p0 + c) : 0.0;
        lp1[q] = p1 ? __ldg(p1 + c) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int m = 4 * h + q;
        const int c = t + FU_T * m;
        if (o0) {
          const double val = v[m].x + lb0[q];
          o0[c] = val;
          const double d = val - lp0[q];
          acc[0] = fma(d, d, acc[0]);
          acc[1] = fma(lp0[q], lp0[q], acc[1]);
          acc[2] += isfinite(val) ? 0.0 : 1.0;
        }
        if (o1) {
          const double val = v[m].y + lb1[q];
          o1[c] = val;
          const double d = val - lp1[q];
          acc[3] = fma(d, d, acc[3]);
          acc[4] = fma(lp1[q], lp1[q], acc[4]);
          acc[5] += isfinite(val) ? 0.0 : 1.0;
        }
      }
    }
  }
  block_sum<6>(acc, s_red);
  if (threadIdx.x == 0) {
    double* dst = a.partials + ((long long)p * FU_CL + rank) * 6;
#pragma unroll
    for (int i = 0; i < 6; ++i) dst[i] = acc[i];
  }
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + p, FU_CL, &s_last);
  double tot[6];
  if (lastb) gather_partials<6>(a.partials + (long long)p * FU_CL * 6, FU_CL, tot, s_red);
  if (lastb && threadIdx.x == 0) {
    if (a0) record_step(a.st[b0], b0, tot[0], tot[1], tot[2], a.S, a.ctl, a.tr);
    if (a1) record_step(a.st[b1], b1, tot[3], tot[4], tot[5], a.S, a.ctl, a.tr);
  }
}

template <int DK>
static void fused_t(const FusedArgs& a, int npairs, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_fused_step<DK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    done = true;
  }
  k_fused_step<DK><<<dim3(FU_CL, npairs), FU_THREADS, fused_smem(a.dn), s>>>(a);
}

void launch_fused_step(const FusedArgs& a, int npairs, cudaStream_t s) {
  switch (a.dn.kind) {
    case DN_MEDIAN3: fused_t<DN_MEDIAN3>(a, npairs, s); break;
    case DN_CONV: fused_t<DN_CONV>(a, npairs, s); break;
    default: fused_t<DN_IDENTITY>(a, npairs, s); break;
  }
}

}  // namespace redve
