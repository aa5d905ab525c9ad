// Probe: the PatchWeighted vector sweep rebuilt feature by feature on top of the bare plane read of
// pw_stream_probe.cu (interior tiles only, no parity: timing of what each ingredient costs).
//   F_FMA     fp32 -> fp64 convert + DFMA into 4 accumulators (v = a register constant)
//   F_SMEM    v from the shared D tile (prologue: tile load + barrier), k-major reads like the product kernel
//   F_MIRROR  the mirrored weights w0_k(p - o_k) spliced from two aligned 16-byte loads
//   F_STORE   D_out = d / sqrt(d S)
//   F_NOPRO   (with F_SMEM) skip the prologue: shared reads of an unfilled tile, no barrier
//   F_NOLDS   (with F_SMEM) prologue + barrier, but v stays a register constant
//   F_FASTEPI D_out = d * rsqrt(d S) by MUFU.RSQ64H + two Newton steps
//   F_ROWMAJOR the search window row by row: VW + 6 values of v per row in registers (16-byte shared loads)
//   F_ICVT    fp32 -> fp64 by two integer multiply-adds (positive normal weights) instead of F2F on the XU pipe
//   F_SHFL    the second mirrored vector taken from lane + 1's first one (shuffles; lane 31 loads it)
//   F_SWZ     D tile columns stored as 4 interleaved sub-rows (column c at (c & 3) * 34 + (c >> 2)): lane-consecutive, conflict-free v reads
//   F_HOIST   the first offset's three plane vectors requested before the prologue's wait + barrier
//   F_DSMEM   the epilogue's d taken from the tile centre instead of global memory
//   F_ASYNC   prologue by cp.async (16-byte pieces of the aligned tile interior skipped: 8-byte LDGSTS)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pw_sweep_probe tools/pw_sweep_probe.cu && /tmp/pw_sweep_probe
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
constexpr int SR = 3, SIDE = 7, NP = 24, VW = 4, TW = 128, TH = 8, X = TW + 2 * SR, Y = TH + 2 * SR;
enum { F_FMA = 1, F_SMEM = 2, F_MIRROR = 4, F_STORE = 8, F_NOPRO = 16, F_NOLDS = 32, F_FASTEPI = 64, F_ROWMAJOR = 128, F_ASYNC = 256, F_ICVT = 512, F_SHFL = 1024, F_SWZ = 2048, F_HOIST = 4096, F_DSMEM = 8192 };
__host__ __device__ constexpr int DI(int k) { return ((SIDE * SIDE + 1) / 2 + k) / SIDE - SR; }
__host__ __device__ constexpr int DJ(int k) { return ((SIDE * SIDE + 1) / 2 + k) % SIDE - SR; }
__host__ __device__ constexpr int QB(int q) { return q >= 0 ? q / VW : -((-q + VW - 1) / VW); }
__host__ __device__ constexpr int QR(int q) { return q - VW * QB(q); }
union WV { int4 raw; float e[4]; };
constexpr int XS = 136;  // swizzled row stride (4 sub-rows of 34)
template <int F>
__device__ __forceinline__ int vidx(int row, int col) {
  return (F & F_SWZ) ? row * XS + (col & 3) * 34 + (col >> 2) : row * X + col;
}
template <int F>
__device__ __forceinline__ double cvt(float x) {
  if (F & F_ICVT) {
    const unsigned u = __float_as_uint(x);
    return __hiloint2double((int)(__umulhi(u, 0x20000000u) + 0x38000000u), (int)(u << 29));
  }
  return (double)x;
}
__device__ __forceinline__ double fast_rsqrt(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));  // MUFU.RSQ64H: ~20 bits
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
template <int F, int MINB>
__global__ void __launch_bounds__(256, MINB) k_sweep(const float* __restrict__ w, const double* __restrict__ Din,
                                                     double* Dout, int H, int W) {
  extern __shared__ double vs[];
  const int lane = threadIdx.x & 31, oi = threadIdx.x >> 5;
  const int i0 = (blockIdx.y + 1) * TH, j0 = (blockIdx.x + 1) * TW;
  const long long N = (long long)H * W;
  WV h_wp, h_lo, h_hi;
  if (F & F_HOIST) {
    const long long oo = (long long)(i0 + oi) * W + j0 + VW * lane;
    h_wp.raw = __ldg(reinterpret_cast<const int4*>(w + oo));
    const long long om = oo - (long long)DI(0) * W + VW * QB(-DJ(0));
    h_lo.raw = __ldg(reinterpret_cast<const int4*>(w + om));
    h_hi.raw = __ldg(reinterpret_cast<const int4*>(w + om + VW));
  }
  if ((F & F_SMEM) && !(F & F_NOPRO)) {
    for (int idx = threadIdx.x; idx < Y * X; idx += 256) {
      const int ti = idx / X, tj = idx - ti * X;
      const double* src = Din + (long long)(i0 - SR + ti) * W + (j0 - SR + tj);
      if (F & F_ASYNC) {
        const unsigned dst = (unsigned)__cvta_generic_to_shared(vs + vidx<F>(ti, tj));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src));
      } else {
        vs[vidx<F>(ti, tj)] = __ldg(src);
      }
    }
    if (F & F_ASYNC) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  const int gi = i0 + oi, gj = j0 + VW * lane, ci = oi + SR, cj = VW * lane + SR;
  const long long o = (long long)gi * W + gj;
  double S[VW];
#pragma unroll
  for (int t = 0; t < VW; ++t) S[t] = (F & F_SMEM) ? vs[vidx<F>(ci, cj + t)] : 1.0;
  float facc = 0.f;
  if (F & F_ROWMAJOR) {
#pragma unroll
    for (int r = -SR; r <= SR; ++r) {
      double v[VW + 2 * SR];
      const double2* vrow = reinterpret_cast<const double2*>(vs + (ci + r) * X + VW * lane);
#pragma unroll
      for (int c = 0; c < (VW + 2 * SR) / 2; ++c) { const double2 t2 = vrow[c]; v[2 * c] = t2.x; v[2 * c + 1] = t2.y; }
#pragma unroll
      for (int dj = -SR; dj <= SR; ++dj) {
        if (r == 0 && dj <= 0) continue;
        if (r >= 0) {
          const int k = (r + SR) * SIDE + dj + SR - (SIDE * SIDE + 1) / 2;
          WV wp; wp.raw = __ldg(reinterpret_cast<const int4*>(w + (long long)k * N + o));
#pragma unroll
          for (int t = 0; t < VW; ++t) S[t] = fma(cvt<F>(wp.e[t]), v[t + dj + SR], S[t]);
        }
        if (r <= 0) {
          const int di = -r, dj2 = (r == 0) ? dj : -dj;
          const int k = (di + SR) * SIDE + dj2 + SR - (SIDE * SIDE + 1) / 2;
          const long long om = (long long)k * N + o - (long long)di * W + VW * QB(-dj2);
          WV lo, hi;
          lo.raw = __ldg(reinterpret_cast<const int4*>(w + om));
          if (QR(-dj2) != 0) {
            if (F & F_SHFL) {
#pragma unroll
              for (int e = 0; e < QR(-dj2); ++e) hi.e[e] = __shfl_down_sync(0xffffffffu, lo.e[e], 1);
              if (lane == 31) hi.raw = __ldg(reinterpret_cast<const int4*>(w + om + VW));
            } else hi.raw = __ldg(reinterpret_cast<const int4*>(w + om + VW));
          } else hi.raw = lo.raw;
#pragma unroll
          for (int t = 0; t < VW; ++t) {
            const int u = t + QR(-dj2);
            const double wm = cvt<F>(u < VW ? lo.e[u < VW ? u : 0] : hi.e[u >= VW ? u - VW : 0]);
            S[t] = fma(wm, v[t - dj2 + SR], S[t]);
          }
        }
      }
    }
  } else
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    constexpr int dummy = 0; (void)dummy;
    const int di = DI(k), dj = DJ(k);
    const float* wk = w + (long long)k * N;
    WV wp, lo, hi;
    if ((F & F_HOIST) && k == 0) { wp = h_wp; lo = h_lo; hi = h_hi; } else {
    wp.raw = __ldg(reinterpret_cast<const int4*>(wk + o));
    if (F & F_MIRROR) {
      const long long om = o - (long long)di * W + VW * QB(-dj);
      lo.raw = __ldg(reinterpret_cast<const int4*>(wk + om));
      if (QR(-dj) != 0) {
        if (F & F_SHFL) {
#pragma unroll
          for (int e = 0; e < QR(-dj); ++e) hi.e[e] = __shfl_down_sync(0xffffffffu, lo.e[e], 1);
          if (lane == 31) hi.raw = __ldg(reinterpret_cast<const int4*>(wk + om + VW));
        } else hi.raw = __ldg(reinterpret_cast<const int4*>(wk + om + VW));
      } else hi.raw = lo.raw;
    }
    }
    if (F & F_FMA) {
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        const double vp = ((F & F_SMEM) && !(F & F_NOLDS)) ? vs[vidx<F>(ci + di, cj + t + dj)] : 1.25;
        S[t] = fma(cvt<F>(wp.e[t]), vp, S[t]);
        if (F & F_MIRROR) {
          const int u = t + QR(-dj);
          const double wm = cvt<F>(u < VW ? lo.e[u < VW ? u : 0] : hi.e[u >= VW ? u - VW : 0]);
          const double vm = ((F & F_SMEM) && !(F & F_NOLDS)) ? vs[vidx<F>(ci - di, cj + t - dj)] : 0.75;
          S[t] = fma(wm, vm, S[t]);
        }
      }
    } else {
      facc += wp.e[0] + wp.e[1] + wp.e[2] + wp.e[3];
      if (F & F_MIRROR) facc += lo.e[0] + lo.e[3] + hi.e[0] + hi.e[3];
    }
  }
  if (F & F_STORE) {
#pragma unroll
    for (int t = 0; t < VW; ++t) {
      const double d = (F & F_DSMEM) ? vs[vidx<F>(ci, cj + t)] : Din[o + t];
      const double a = d * S[t] + (double)facc;
      Dout[o + t] = (F & F_FASTEPI) ? d * fast_rsqrt(a) : d / sqrt(a);
    }
  } else if (S[0] + S[1] + S[2] + S[3] + (double)facc == 12345.678) Dout[0] = S[0];
}
template <class Fn>
static float timeit(Fn f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f();
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}
static float* g_w; static double *g_d0, *g_d1; static int g_H, g_W;

// Persistent form: one CTA per residency slot walks tiles; the D tile of the next tile arrives by cp.async while
// this tile's offsets run, the epilogue takes d from the tile's centre.
template <int F, int MINB>
__global__ void __launch_bounds__(256, MINB) k_sweep_p(const float* __restrict__ w, const double* __restrict__ Din,
                                                       double* Dout, int H, int W, int ntx, int nty) {
  extern __shared__ double vsb[];
  const int lane = threadIdx.x & 31, oi = threadIdx.x >> 5;
  const long long N = (long long)H * W;
  const int ntile = ntx * nty;
  auto issue = [&](int tile, double* vs) {
    const int i0 = (tile / ntx + 1) * TH, j0 = (tile % ntx + 1) * TW;
    for (int idx = threadIdx.x; idx < Y * X; idx += 256) {
      const int ti = idx / X, tj = idx - ti * X;
      const double* src = Din + (long long)(i0 - SR + ti) * W + (j0 - SR + tj);
      const unsigned dst = (unsigned)__cvta_generic_to_shared(vs + idx);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int tile = blockIdx.x, buf = 0;
  if (tile < ntile) issue(tile, vsb);
  for (; tile < ntile; tile += gridDim.x, buf ^= 1) {
    const double* vs = vsb + buf * (X * Y);
    if (tile + (int)gridDim.x < ntile) {
      issue(tile + gridDim.x, vsb + (buf ^ 1) * (X * Y));
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int i0 = (tile / ntx + 1) * TH, j0 = (tile % ntx + 1) * TW;
    const int gi = i0 + oi, gj = j0 + VW * lane, ci = oi + SR, cj = VW * lane + SR;
    const long long o = (long long)gi * W + gj;
    double S[VW];
#pragma unroll
    for (int t = 0; t < VW; ++t) S[t] = vs[ci * X + cj + t];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int di = DI(k), dj = DJ(k);
      const float* wk = w + (long long)k * N;
      WV wp, lo, hi;
      wp.raw = __ldg(reinterpret_cast<const int4*>(wk + o));
      const long long om = o - (long long)di * W + VW * QB(-dj);
      lo.raw = __ldg(reinterpret_cast<const int4*>(wk + om));
      if (QR(-dj) != 0) {
        if (F & F_SHFL) {
#pragma unroll
          for (int e = 0; e < QR(-dj); ++e) hi.e[e] = __shfl_down_sync(0xffffffffu, lo.e[e], 1);
          if (lane == 31) hi.raw = __ldg(reinterpret_cast<const int4*>(wk + om + VW));
        } else hi.raw = __ldg(reinterpret_cast<const int4*>(wk + om + VW));
      } else hi.raw = lo.raw;
#pragma unroll
      for (int t = 0; t < VW; ++t) {
        S[t] = fma(cvt<F>(wp.e[t]), vs[(ci + di) * X + cj + t + dj], S[t]);
        const int u = t + QR(-dj);
        const double wm = cvt<F>(u < VW ? lo.e[u < VW ? u : 0] : hi.e[u >= VW ? u - VW : 0]);
        S[t] = fma(wm, vs[(ci - di) * X + cj + t - dj], S[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < VW; ++t) {
      const double d = vs[ci * X + cj + t];
      const double a = d * S[t];
      Dout[o + t] = (F & F_FASTEPI) ? d * fast_rsqrt(a) : d / sqrt(a);
    }
    __syncthreads();
  }
}
template <int F, int MINB>
static void runp(const char* name) {
  const int ntx = g_W / TW - 2, nty = g_H / TH - 2;
  const size_t sm = 2 * sizeof(double) * X * Y;
  const float t = timeit([&] { k_sweep_p<F, MINB><<<148 * MINB, 256, sm>>>(g_w, g_d0, g_d1, g_H, g_W, ntx, nty); });
  const double gb = (double)NP * ntx * nty * TW * TH * 4 / 1e9;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_sweep_p<F, MINB>);
  printf("%-34s minb %d regs %3d  %7.3f ms  %7.1f GB/s (planes)  %s\n", name, MINB, fa.numRegs, t, gb / t * 1e3,
         cudaGetErrorString(cudaGetLastError()));
}
#define RUNP(F, name) runp<F, 6>(name); runp<F, 5>(name); runp<F, 4>(name); runp<F, 3>(name);

template <int F, int MINB>
static void run(const char* name) {
  dim3 grid(g_W / TW - 2, g_H / TH - 2);
  const size_t sm = sizeof(double) * XS * Y;
  const float t = timeit([&] { k_sweep<F, MINB><<<grid, 256, sm>>>(g_w, g_d0, g_d1, g_H, g_W); });
  const double gb = (double)NP * grid.x * grid.y * TW * TH * 4 / 1e9;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_sweep<F, MINB>);
  printf("%-34s minb %d regs %3d  %7.3f ms  %7.1f GB/s (planes)  %s\n", name, MINB, fa.numRegs, t, gb / t * 1e3,
         cudaGetErrorString(cudaGetLastError()));
}
#define RUNALL(F, name) run<F, 5>(name); run<F, 4>(name); run<F, 3>(name); run<F, 2>(name);
int main(int argc, char** argv) {
  g_H = argc > 2 ? atoi(argv[1]) : 8192; g_W = argc > 2 ? atoi(argv[2]) : 8192;
  const long long N = (long long)g_H * g_W;
  cudaMalloc(&g_w, NP * N * 4); cudaMalloc(&g_d0, N * 8); cudaMalloc(&g_d1, N * 8);
  cudaMemset(g_w, 0x3c, NP * N * 4);  // ~0.0115 per weight
  cudaMemset(g_d0, 0x3f, N * 8);
  constexpr int FULL = F_FMA | F_MIRROR | F_SMEM | F_STORE;
#define RUN4(F, name) run<F, 6>(name); run<F, 5>(name); run<F, 4>(name); run<F, 3>(name);
  constexpr int BEST = FULL | F_SWZ | F_FASTEPI | F_ICVT | F_SHFL | F_ASYNC;
  RUN4(BEST, "best so far")
  RUN4(BEST | F_DSMEM, "best + d from tile")
  RUN4(BEST | F_HOIST, "best + hoist")
  RUN4(BEST | F_HOIST | F_DSMEM, "best + hoist + d from tile")
  RUN4((BEST | F_HOIST | F_DSMEM) & ~F_SHFL, "  ... without shfl")
  RUN4((BEST | F_HOIST | F_DSMEM) & ~F_ICVT, "  ... without icvt")
  RUN4((BEST | F_HOIST | F_DSMEM) & ~F_FASTEPI, "  ... without fast epi")
  RUN4((BEST | F_HOIST | F_DSMEM) & ~F_SWZ, "  ... without swizzle")
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
