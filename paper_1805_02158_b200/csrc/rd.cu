// Seeded reaction-diffusion (filter-bank) denoiser for BASELINE.json configs[3]:
//   f(x) = x - tau * sum_i  k_i (*) phi_i( k_i (x) x ),   phi_i(z) = z / (1 + z^2 / s_i^2)
// ((x) = periodic correlation, (*) = its adjoint, the periodic convolution).
// One fused tiled kernel: x tile with halo 2r, every filter's influence
// response phi_i on the tile with halo r kept in shared memory, then the
// adjoint filters back -- x is read once and f written once.
// No reference implementation exists: the in-repo
// oracle is oracle/extras.py FilterBank ("parity unpinned").
#include "kernels.cuh"
#include "rd.cuh"

namespace redve {

extern __shared__ __align__(16) unsigned char r_smem[];

constexpr int RD_T = 32;

__global__ void __launch_bounds__(256) k_rd_denoise(RdArgs a) {
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W, fs = a.fs, r = fs / 2, nf = a.nf;
  const int X = RD_T + 4 * r;  // x tile edge
  const int P = RD_T + 2 * r;  // phi tile edge
  double* ks = reinterpret_cast<double*>(r_smem);
  double* sc = ks + nf * fs * fs;
  double* xs = sc + nf;
  double* ph = xs + X * X;
  for (int i = threadIdx.x; i < nf * fs * fs; i += blockDim.x) ks[i] = a.filters[i];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) sc[i] = 1.0 / (a.scales[i] * a.scales[i]);
  const int i0 = blockIdx.y * RD_T, j0 = blockIdx.x * RD_T;
  const double* x = a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < X * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    xs[idx] = __ldg(x + (long long)wrap(i0 - 2 * r + ti, H) * W + wrap(j0 - 2 * r + tj, W));
  }
  __syncthreads();
  // phi_i over the tile + halo r: z(q) = sum_ab k[a][b] x(q + (a-r, b-r))
  for (int idx = threadIdx.x; idx < nf * P * P; idx += blockDim.x) {
    const int f = idx / (P * P), rem = idx - f * P * P;
    const int pi = rem / P, pj = rem - pi * P;
    const double* kf = ks + f * fs * fs;
    double z = 0.0;
    for (int ta = 0; ta < fs; ++ta)
      for (int tb = 0; tb < fs; ++tb) z = fma(kf[ta * fs + tb], xs[(pi + ta) * X + (pj + tb)], z);
    ph[idx] = z / fma(z * z, sc[f], 1.0);
  }
  __syncthreads();
  const long long N = (long long)H * W;
  for (int idx = threadIdx.x; idx < RD_T * RD_T; idx += blockDim.x) {
    const int oi = idx / RD_T, oj = idx - oi * RD_T;
    const int gi = i0 + oi, gj = j0 + oj;
    if (gi >= H || gj >= W) continue;
    // adjoint: sum_ab k[a][b] phi(p - (a-r, b-r))
    double acc = 0.0;
    for (int f = 0; f < nf; ++f) {
      const double* kf = ks + f * fs * fs;
      const double* pf = ph + f * P * P;
      for (int ta = 0; ta < fs; ++ta)
        for (int tb = 0; tb < fs; ++tb)
          acc = fma(kf[ta * fs + tb], pf[(oi + 2 * r - ta) * P + (oj + 2 * r - tb)], acc);
    }
    const double xv = xs[(oi + 2 * r) * X + (oj + 2 * r)];
    a.out[(long long)b * N + (long long)gi * W + gj] = fma(-a.tau, acc, xv);
  }
}

// Register-blocked specialisation for FS x FS filters: per filter, the
// influence response on the tile + halo r is formed by column strips of
// RD_S1 rows (each loaded x column segment feeds FS*RD_S1 FMAs), written to
// a double-buffered shared tile, and the adjoint filter is accumulated into
// RD_S2-row output strips held in registers across all filters.
constexpr int RD_S1 = 6, RD_S2 = 4;

template <int FS>
__global__ void __launch_bounds__(256) k_rd_fast(RdArgs a) {
  constexpr int R = FS / 2, X = RD_T + 4 * R, P = RD_T + 2 * R;
  constexpr int NS1 = (P + RD_S1 - 1) / RD_S1;
  static_assert(RD_T * RD_T == 256 * RD_S2, "one output strip per thread");
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W, nf = a.nf;
  double* ks = reinterpret_cast<double*>(r_smem);
  double* sc = ks + nf * FS * FS;
  double* xs = sc + nf;
  double* ph = xs + X * X;  // [2][P][P]
  for (int i = threadIdx.x; i < nf * FS * FS; i += blockDim.x) ks[i] = a.filters[i];
  for (int i = threadIdx.x; i < nf; i += blockDim.x) sc[i] = 1.0 / (a.scales[i] * a.scales[i]);
  const int i0 = blockIdx.y * RD_T, j0 = blockIdx.x * RD_T;
  const double* x = a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < X * X; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    xs[idx] = __ldg(x + (long long)wrap_fast(i0 - 2 * R + ti, H) * W + wrap_fast(j0 - 2 * R + tj, W));
  }
  __syncthreads();
  const int t = threadIdx.x;
  const bool p1 = t < NS1 * P;
  const int pc = t % P, pr0 = (t / P) * RD_S1;
  const int oc = t & (RD_T - 1), or0 = (t >> 5) * RD_S2;
  double acc[RD_S2];
#pragma unroll
  for (int m = 0; m < RD_S2; ++m) acc[m] = 0.0;
  for (int f = 0; f < nf; ++f) {
    double* phb = ph + (f & 1) * P * P;
    const double* kf = ks + f * FS * FS;
    if (p1) {  // phi_f(q) = z / (1 + z^2/s^2), z = sum_ab k[a][b] x(q + (a-r, b-r))
      double z[RD_S1];
#pragma unroll
      for (int m = 0; m < RD_S1; ++m) z[m] = 0.0;
#pragma unroll
      for (int tb = 0; tb < FS; ++tb) {
        double v[RD_S1 + FS - 1];
#pragma unroll
        for (int u = 0; u < RD_S1 + FS - 1; ++u)
          v[u] = (P % RD_S1 == 0 || pr0 + u < X) ? xs[(pr0 + u) * X + pc + tb] : 0.0;
#pragma unroll
        for (int ta = 0; ta < FS; ++ta) {
          const double kk = kf[ta * FS + tb];
#pragma unroll
          for (int m = 0; m < RD_S1; ++m) z[m] = fma(kk, v[m + ta], z[m]);
        }
      }
      const double sf = sc[f];
#pragma unroll
      for (int m = 0; m < RD_S1; ++m)
        if (P % RD_S1 == 0 || pr0 + m < P) phb[(pr0 + m) * P + pc] = z[m] / fma(z[m] * z[m], sf, 1.0);
    }
    __syncthreads();
    // adjoint: acc(p) += sum_ab k[a][b] phi(p - (a-r, b-r))
#pragma unroll
    for (int tb = 0; tb < FS; ++tb) {
      double v[RD_S2 + FS - 1];
#pragma unroll
      for (int u = 0; u < RD_S2 + FS - 1; ++u) v[u] = phb[(or0 + u) * P + oc + 2 * R - tb];
#pragma unroll
      for (int ta = 0; ta < FS; ++ta) {
        const double kk = kf[ta * FS + tb];
#pragma unroll
        for (int m = 0; m < RD_S2; ++m) acc[m] = fma(kk, v[m + 2 * R - ta], acc[m]);
      }
    }
  }
  const long long N = (long long)H * W;
  const int gj = j0 + oc;
#pragma unroll
  for (int m = 0; m < RD_S2; ++m) {
    const int gi = i0 + or0 + m;
    if (gi >= H || gj >= W) continue;
    const double xv = xs[(or0 + m + 2 * R) * X + (oc + 2 * R)];
    a.out[(long long)b * N + (long long)gi * W + gj] = fma(-a.tau, acc[m], xv);
  }
}

// configs[3] shape of the stage (8 filters of 5x5): taps and scales in
// constant memory (uniform operands of the FMAs, no shared loads), a 64 x 32
// output tile, influence strips of 12 rows and adjoint strips of 8 rows so
// every loaded column value feeds 5 x strip FMAs.
constexpr int RB_NF = 8, RB_FS = 5, RB_TW = 64, RB_TH = 32, RB_S1 = 12, RB_S2 = 8;
__constant__ double c_rb_taps[RB_NF * RB_FS * RB_FS];

__global__ void __launch_bounds__(256) k_rd_bank8(RdArgs a) {
  constexpr int R = RB_FS / 2;
  constexpr int X = RB_TW + 4 * R, XH = RB_TH + 4 * R;  // x tile
  constexpr int PW = RB_TW + 2 * R, PH = RB_TH + 2 * R;  // influence tile
  constexpr int NS1 = PH / RB_S1;                       // 3 strips x 68 columns
  static_assert(PH % RB_S1 == 0 && RB_TH % RB_S2 == 0, "strip shapes");
  static_assert((RB_TH / RB_S2) * RB_TW == 256, "one adjoint strip per thread");
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W;
  __shared__ double s_isc[RB_NF];
  if (threadIdx.x < RB_NF) s_isc[threadIdx.x] = 1.0 / (a.scales[threadIdx.x] * a.scales[threadIdx.x]);
  double* xs = reinterpret_cast<double*>(r_smem);
  double* ph = xs + X * XH;  // [2][PH][PW]
  const int i0 = blockIdx.y * RB_TH, j0 = blockIdx.x * RB_TW;
  const double* x = a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < X * XH; idx += blockDim.x) {
    const int ti = idx / X, tj = idx - ti * X;
    xs[idx] = __ldg(x + (long long)wrap_fast(i0 - 2 * R + ti, H) * W + wrap_fast(j0 - 2 * R + tj, W));
  }
  __syncthreads();
  const int t = threadIdx.x;
  const bool p1 = t < NS1 * PW;
  const int pc = t % PW, pr0 = (t / PW) * RB_S1;
  const int oc = t & (RB_TW - 1), or0 = (t / RB_TW) * RB_S2;
  double acc[RB_S2];
#pragma unroll
  for (int m = 0; m < RB_S2; ++m) acc[m] = 0.0;
#pragma unroll
  for (int f = 0; f < RB_NF; ++f) {
    double* phb = ph + (f & 1) * PH * PW;
    if (p1) {
      double z[RB_S1];
#pragma unroll
      for (int m = 0; m < RB_S1; ++m) z[m] = 0.0;
#pragma unroll
      for (int tb = 0; tb < RB_FS; ++tb) {
        double v[RB_S1 + RB_FS - 1];
#pragma unroll
        for (int u = 0; u < RB_S1 + RB_FS - 1; ++u) v[u] = xs[(pr0 + u) * X + pc + tb];
#pragma unroll
        for (int ta = 0; ta < RB_FS; ++ta) {
          const double kk = c_rb_taps[(f * RB_FS + ta) * RB_FS + tb];
#pragma unroll
          for (int m = 0; m < RB_S1; ++m) z[m] = fma(kk, v[m + ta], z[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < RB_S1; ++m)
        phb[(pr0 + m) * PW + pc] = z[m] / fma(z[m] * z[m], s_isc[f], 1.0);
    }
    __syncthreads();
#pragma unroll
    for (int tb = 0; tb < RB_FS; ++tb) {
      double v[RB_S2 + RB_FS - 1];
#pragma unroll
      for (int u = 0; u < RB_S2 + RB_FS - 1; ++u) v[u] = phb[(or0 + u) * PW + oc + 2 * R - tb];
#pragma unroll
      for (int ta = 0; ta < RB_FS; ++ta) {
        const double kk = c_rb_taps[(f * RB_FS + ta) * RB_FS + tb];
#pragma unroll
        for (int m = 0; m < RB_S2; ++m) acc[m] = fma(kk, v[m + 2 * R - ta], acc[m]);
      }
    }
  }
  const long long N = (long long)H * W;
  const int gj = j0 + oc;
#pragma unroll
  for (int m = 0; m < RB_S2; ++m) {
    const int gi = i0 + or0 + m;
    if (gi >= H || gj >= W) continue;
    const double xv = xs[(or0 + m + 2 * R) * X + (oc + 2 * R)];
    a.out[(long long)b * N + (long long)gi * W + gj] = fma(-a.tau, acc[m], xv);
  }
}

// Wide-tile variant (the default): 64 x 64 outputs per CTA, every thread a
// 2-column block (influence: 2 x 10 rows, adjoint: 2 x 8 rows), so each
// 16-byte shared-memory read feeds two output columns.  ncu on k_rd_bank8:
// FP64 pipe 67% with shared-memory wavefronts at 70% (LDS.64, 2.4 bytes per
// FMA) and 52 of 256 threads idle in the influence pass; here 1.4 bytes per
// FMA and 238 / 256 threads busy in the influence pass.
constexpr int RW_T = 64, RW_S1 = 10, RW_S2 = 8;
constexpr int RW_PW = RW_T + 4, RW_PH = 7 * RW_S1;   // influence tile (68 used rows of 70)
constexpr int RW_X = RW_T + 8, RW_XH = RW_PH + 4;    // x tile: 72 columns x 74 rows
constexpr size_t rw_smem() { return sizeof(double) * ((size_t)RW_X * RW_XH + (size_t)RW_PH * RW_PW); }

// 1/d for d >= 1 (the influence denominator 1 + z^2/s^2): the hardware
// estimate refined by two Newton steps (error 2^-88 before rounding), then one
// rounding in the product -- within an ulp of the correctly rounded quotient,
// at ~6 FP64 instructions instead of the division's ~10.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

__global__ void __launch_bounds__(256, 2) k_rd_bank8w(RdArgs a) {
  constexpr int FS = RB_FS, NF = RB_NF;
  const int b = blockIdx.z;
  if (!takes_step(a.st[b], a.phase)) return;
  const int H = a.H, W = a.W;
  __shared__ double s_isc[NF];
  if (threadIdx.x < NF) s_isc[threadIdx.x] = 1.0 / (a.scales[threadIdx.x] * a.scales[threadIdx.x]);
  double* xs = reinterpret_cast<double*>(r_smem);  // rows i0-4 .., columns j0-4 ..
  double* ph = xs + RW_X * RW_XH;                   // rows i0-2 .., columns j0-2 ..
  const int i0 = blockIdx.y * RW_T, j0 = blockIdx.x * RW_T;
  const double* x = a.xin.at(b, a.st);
  for (int idx = threadIdx.x; idx < RW_X * RW_XH; idx += blockDim.x) {
    const int ti = idx / RW_X, tj = idx - ti * RW_X;
    xs[idx] = __ldg(x + (long long)wrap(i0 - 4 + ti, H) * W + wrap(j0 - 4 + tj, W));
  }
  const int t = threadIdx.x;
  const bool p1 = t < (RW_PW / 2) * (RW_PH / RW_S1);
  const int pc = 2 * (t % (RW_PW / 2)), pr0 = (t / (RW_PW / 2)) * RW_S1;
  const int oc = 2 * (t & 31), or0 = (t >> 5) * RW_S2;
  double acc[RW_S2][2];
#pragma unroll
  for (int m = 0; m < RW_S2; ++m) acc[m][0] = acc[m][1] = 0.0;
  __syncthreads();
#pragma unroll 1
  for (int f = 0; f < NF; ++f) {
    const double* kf = c_rb_taps + f * FS * FS;
    if (p1) {  // phi over influence rows pr0.., columns pc, pc+1: x rows pr0+ta, columns pc+tb
      double z[RW_S1][2];
#pragma unroll
      for (int m = 0; m < RW_S1; ++m) z[m][0] = z[m][1] = 0.0;
#pragma unroll
      for (int u = 0; u < RW_S1 + FS - 1; ++u) {
        double xv[6];
        const double2* row = reinterpret_cast<const double2*>(xs + (pr0 + u) * RW_X + pc);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const double2 v = row[q];
          xv[2 * q] = v.x;
          xv[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int m = 0; m < RW_S1; ++m) {
          const int ta = u - m;
          if (ta < 0 || ta >= FS) continue;
#pragma unroll
          for (int tb = 0; tb < FS; ++tb) {
            const double kk = kf[ta * FS + tb];
            z[m][0] = fma(kk, xv[tb], z[m][0]);
            z[m][1] = fma(kk, xv[tb + 1], z[m][1]);
          }
        }
      }
      const double isc = s_isc[f];
#pragma unroll
      for (int m = 0; m < RW_S1; ++m) {
        double2 o;
        o.x = z[m][0] * rcp_nr(fma(z[m][0] * z[m][0], isc, 1.0));
        o.y = z[m][1] * rcp_nr(fma(z[m][1] * z[m][1], isc, 1.0));
        *reinterpret_cast<double2*>(ph + (pr0 + m) * RW_PW + pc) = o;
      }
    }
    __syncthreads();
    // adjoint: out(r, c) += k[ta][tb] phi(r + 2 - ta, c + 2 - tb); phi rows or0 + m + 4 - ta,
    // columns oc + 4 - tb (+1 for the second column)
#pragma unroll
    for (int u = 0; u < RW_S2 + FS - 1; ++u) {
      double pv[6];
      const double2* row = reinterpret_cast<const double2*>(ph + (or0 + u) * RW_PW + oc);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double2 v = row[q];
        pv[2 * q] = v.x;
        pv[2 * q + 1] = v.y;
      }
#pragma unroll
      for (int m = 0; m < RW_S2; ++m) {
        const int ta = m + 4 - u;
        if (ta < 0 || ta >= FS) continue;
#pragma unroll
        for (int tb = 0; tb < FS; ++tb) {
          const double kk = kf[ta * FS + tb];
          acc[m][0] = fma(kk, pv[4 - tb], acc[m][0]);
          acc[m][1] = fma(kk, pv[5 - tb], acc[m][1]);
        }
      }
    }
    __syncthreads();  // phi is overwritten by the next filter
  }
  const long long N = (long long)H * W;
#pragma unroll
  for (int m = 0; m < RW_S2; ++m) {
    const int gi = i0 + or0 + m;
    if (gi >= H) break;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int gj = j0 + oc + c;
      if (gj >= W) continue;
      const double xv = xs[(or0 + m + 4) * RW_X + (oc + c + 4)];
      a.out[(long long)b * N + (long long)gi * W + gj] = fma(-a.tau, acc[m][c], xv);
    }
  }
}

static bool launch_rd_bank8(const RdArgs& a, cudaStream_t s) {
  if (a.nf != RB_NF || a.fs != RB_FS) return false;
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_rd_bank8, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = true;
  }
  // taps into constant memory (stream-ordered; a memcpy node under graph capture)
  cudaMemcpyToSymbolAsync(c_rb_taps, a.filters, sizeof(double) * RB_NF * RB_FS * RB_FS, 0,
                          cudaMemcpyDeviceToDevice, s);
  constexpr int R = RB_FS / 2;
  const size_t smem = sizeof(double) * ((size_t)(RB_TW + 4 * R) * (RB_TH + 4 * R) +
                                        2 * (size_t)(RB_TW + 2 * R) * (RB_TH + 2 * R));
  const char* e = getenv("REDVE_FB_WIDE");
  if (!(e && e[0] == '0')) {
    static bool wdone = false;
    if (!wdone) {
      cudaFuncSetAttribute(k_rd_bank8w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rw_smem());
      wdone = true;
    }
    dim3 gw((a.W + RW_T - 1) / RW_T, (a.H + RW_T - 1) / RW_T, a.B);
    k_rd_bank8w<<<gw, 256, rw_smem(), s>>>(a);
    return true;
  }
  dim3 grid((a.W + RB_TW - 1) / RB_TW, (a.H + RB_TH - 1) / RB_TH, a.B);
  k_rd_bank8<<<grid, 256, smem, s>>>(a);
  return true;
}

template <int FS>
static size_t rd_fast_smem(int nf) {
  constexpr int R = FS / 2, X = RD_T + 4 * R, P = RD_T + 2 * R;
  return sizeof(double) * ((size_t)nf * FS * FS + nf + (size_t)X * X + 2 * (size_t)P * P);
}

size_t rd_smem(int nf, int fs) {
  const int r = fs / 2, X = RD_T + 4 * r, P = RD_T + 2 * r;
  return sizeof(double) * ((size_t)nf * fs * fs + nf + (size_t)X * X + (size_t)nf * P * P);
}

void launch_rd(const RdArgs& a, cudaStream_t s) {
  static bool done = false;
  if (!done) {
    cudaFuncSetAttribute(k_rd_denoise, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_rd_fast<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_rd_fast<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_rd_fast<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = true;
  }
  if (launch_rd_bank8(a, s)) return;
  dim3 grid((a.W + RD_T - 1) / RD_T, (a.H + RD_T - 1) / RD_T, a.B);
  switch (a.fs) {
    case 3: k_rd_fast<3><<<grid, 256, rd_fast_smem<3>(a.nf), s>>>(a); return;
    case 5: k_rd_fast<5><<<grid, 256, rd_fast_smem<5>(a.nf), s>>>(a); return;
    case 7: k_rd_fast<7><<<grid, 256, rd_fast_smem<7>(a.nf), s>>>(a); return;
    default: k_rd_denoise<<<grid, 256, rd_smem(a.nf, a.fs), s>>>(a);
  }
}

}  // namespace redve
