// Line FFT engine for the fused Fourier fixed-point step (fp64, sm_100a).
//
// One "line" (an image row or column) of length L is transformed by T =
// ceil(L/16) threads.  Register contract, identical on entry and exit:
//     v[m] == element (t + T*m) of the line, m < 16  (valid while < L)
// so a kernel can produce the line straight from its own math (denoiser,
// spectral divide) and consume the transform straight into its epilogue
// without extra shared-memory passes.
//
// * L a power of two: Stockham autosort, radix-16 first stage (from the
//   registers), radix-{16,8,4,2} later stages through shared memory, the last
//   stage lands back in registers.  256-point = two radix-16 stages and one
//   shared-memory round trip.
// * any other L: direct O(L^2) DFT from a table (test sizes like 10, 12, 24).
//
// The unnormalised forward kernel is exp(-2 pi i n k / L) (numpy.fft
// convention, imaging.py:100-110); INV uses the conjugate.
#pragma once

#include "common.cuh"

namespace redve {

// exp(-+2 pi i e / 16) * a, folded to constants when e is a compile-time value
template <bool INV>
__device__ __forceinline__ cd rot16(cd a, int e) {
  constexpr double C1 = 0.92387953251128674, S1 = 0.38268343236508978;
  constexpr double H = 0.70710678118654752;
  double c, s;
  switch (e & 15) {
    case 0: return a;
    case 4: return INV ? cd{-a.y, a.x} : cd{a.y, -a.x};
    case 8: return cd{-a.x, -a.y};
    case 12: return INV ? cd{a.y, -a.x} : cd{-a.y, a.x};
    case 1: c = C1; s = S1; break;
    case 2: c = H; s = H; break;
    case 3: c = S1; s = C1; break;
    case 5: c = -S1; s = C1; break;
    case 6: c = -H; s = H; break;
    case 7: c = -C1; s = S1; break;
    case 9: c = -C1; s = -S1; break;
    case 10: c = -H; s = -H; break;
    case 11: c = -S1; s = -C1; break;
    case 13: c = S1; s = -C1; break;
    case 14: c = H; s = -H; break;
    default: c = C1; s = -S1; break;  // 15
  }
  // angle 2 pi e/16 = (c, s); forward multiplies by (c, -s)
  return INV ? cmul(a, cd{c, s}) : cmul(a, cd{c, -s});
}

template <int N, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  static __device__ __forceinline__ void run(cd*) {}
};

template <bool INV>
struct Dft<2, INV> {
  static __device__ __forceinline__ void run(cd* a) {
    cd u = a[0], w = a[1];
    a[0] = u + w;
    a[1] = u - w;
  }
};

template <bool INV>
struct Dft<4, INV> {
  static __device__ __forceinline__ void run(cd* a) {
    cd t0 = a[0] + a[2], t1 = a[0] - a[2], t2 = a[1] + a[3], t3 = a[1] - a[3];
    // forward: X1 = t1 - i t3, X3 = t1 + i t3
    cd it3 = cd{-t3.y, t3.x};  // i * t3
    a[0] = t0 + t2;
    a[2] = t0 - t2;
    if (INV) {
      a[1] = t1 + it3;
      a[3] = t1 - it3;
    } else {
      a[1] = t1 - it3;
      a[3] = t1 + it3;
    }
  }
};

// four-step N = N1*N2: n = N2*n1 + n2, k = k1 + N1*k2
template <int N1, int N2, bool INV>
__device__ __forceinline__ void four_step(cd* a) {
  constexpr int N = N1 * N2;
  cd b[N];
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) {
    cd t[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) t[n1] = a[N2 * n1 + n2];
    Dft<N1, INV>::run(t);
#pragma unroll
    for (int k1 = 0; k1 < N1; ++k1) b[n2 * N1 + k1] = rot16<INV>(t[k1], (n2 * k1) * (16 / N));
  }
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) {
    cd t[N2];
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) t[n2] = b[n2 * N1 + k1];
    Dft<N2, INV>::run(t);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) a[k1 + N1 * k2] = t[k2];
  }
}

template <bool INV>
struct Dft<8, INV> {
  static __device__ __forceinline__ void run(cd* a) { four_step<4, 2, INV>(a); }
};
template <bool INV>
struct Dft<16, INV> {
  static __device__ __forceinline__ void run(cd* a) { four_step<4, 4, INV>(a); }
};

// ------------------------------------------------------------------ layouts
// Row kernels: line-major, +1 pad per 16 elements (conflict-free radix-16 I/O).
struct RowLayout {
  int stride;
  __device__ __forceinline__ int at(int line, int e) const { return line * stride + e + (e >> 4); }
  static REDVE_HD int stride_for(int L) { return L + (L >> 4) + 1; }
};
// Column kernels: element-major, lanes run across lines.
struct ColLayout {
  int lpc;
  __device__ __forceinline__ int at(int line, int e) const { return e * lpc + line; }
};

REDVE_HD bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }
REDVE_HD int threads_per_line(int L) { return (L + 15) / 16; }

// Stockham stage: radix R, Ns = product of previous radices.  Reads either
// the registers (first stage) or shared memory; writes shared memory or the
// registers (last stage).
template <int R, bool INV, class Lay>
__device__ __forceinline__ void stockham_stage(cd (&v)[16], cd* sm, const cd* tw, int L, int T,
                                               int t, int line, int Ns, bool first, bool last,
                                               const Lay& lay) {
  constexpr int NB = 16 / R;  // butterflies per thread
  const int LR = L / R;
  cd a[NB][R];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
    const int k = j & (Ns - 1);  // j mod Ns (Ns is a power of two)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cd x = first ? v[b * R + r] : ld_cd(sm + lay.at(line, j + r * LR));
      if (!first && r > 0 && k != 0) {
        const int e = r * k * (L / (Ns * R));
        cd w = tw[e];
        x = INV ? cmul(x, w) : cmulc(x, w);
      }
      a[b][r] = x;
    }
    Dft<R, INV>::run(a[b]);
  }
  if (!first) __syncthreads();  // everyone has read before anyone writes
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
    const int k = j & (Ns - 1);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (last) {
        v[b + r * NB] = a[b][r];
      } else {
        st_cd(sm + lay.at(line, base + r * Ns), a[b][r]);
      }
    }
  }
  if (!last) __syncthreads();
}

// First stage for L >= 16: thread t holds in[t + T*r] == in[j + r*L/16] (j=t).
template <bool INV, class Lay>
__device__ void line_fft_pow2(cd (&v)[16], cd* sm, const cd* tw, int L, int t, int line,
                              const Lay& lay) {
  const int T = L >> 4;
  if (L < 16) {
    // single thread per line, single radix-L stage
    switch (L) {
      case 1: break;
      case 2: Dft<2, INV>::run(v); break;
      case 4: Dft<4, INV>::run(v); break;
      case 8: Dft<8, INV>::run(v); break;
    }
    return;
  }
  int Ns = 1;
  int rem = L;
  bool first = true;
  while (rem > 1) {
    int R = rem >= 16 ? 16 : rem;
    bool last = (rem == R);
    switch (R) {
      case 16: stockham_stage<16, INV>(v, sm, tw, L, T, t, line, Ns, first, last, lay); break;
      case 8: stockham_stage<8, INV>(v, sm, tw, L, T, t, line, Ns, first, last, lay); break;
      case 4: stockham_stage<4, INV>(v, sm, tw, L, T, t, line, Ns, first, last, lay); break;
      default: stockham_stage<2, INV>(v, sm, tw, L, T, t, line, Ns, first, last, lay); break;
    }
    Ns *= R;
    rem /= R;
    first = false;
  }
}

// Direct DFT for non-power-of-two L (same register contract).
template <bool INV, class Lay>
__device__ void line_dft_direct(cd (&v)[16], cd* sm, const cd* tw, int L, int T, int t,
                                int line, const Lay& lay) {
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    int e = t + T * m;
    if (e < L) st_cd(sm + lay.at(line, e), v[m]);
  }
  __syncthreads();
#pragma unroll 1
  for (int m = 0; m < 16; ++m) {
    int k = t + T * m;
    if (k >= L) break;
    cd acc = cd{0.0, 0.0};
    int idx = 0;
    for (int n = 0; n < L; ++n) {
      cd x = ld_cd(sm + lay.at(line, n));
      cd w = tw[idx];
      acc = acc + (INV ? cmul(x, w) : cmulc(x, w));
      idx += k;
      if (idx >= L) idx -= L;
    }
    v[m] = acc;
  }
  __syncthreads();
}

// Public entry: all threads of the CTA must call it (it synchronises).
template <bool INV, class Lay>
__device__ __forceinline__ void line_fft(cd (&v)[16], cd* sm, const cd* tw, int L, int t, int line,
                                         const Lay& lay) {
  if (is_pow2(L)) {
    line_fft_pow2<INV>(v, sm, tw, L, t, line, lay);
  } else {
    line_dft_direct<INV>(v, sm, tw, L, threads_per_line(L), t, line, lay);
  }
}

// ------------------------------------------------------------------
// Compile-time specialisation (L a power of two, 16 <= L <= 4096): every
// radix, stride and register index is a constant, so the 16 values stay in
// registers without spills.  FIRST_SMEM: the first stage reads its inputs
// from shared memory (the caller stored them with the same layout) instead of
// the registers.
//
// Twiddles come from a stage-major table: stage (NS, R) owns the block
// tws[off + r*NS + k] = W_{NS R}^{r k}, so the lanes of a warp (consecutive
// k) read consecutive entries -- no shared-memory bank conflicts.
constexpr int tw_stage_size(int L) {
  int ns = 16, rem = L / 16, sz = 0;
  while (rem > 1) {
    int R = rem >= 16 ? 16 : rem;
    sz += R * ns;
    ns *= R;
    rem /= R;
  }
  return sz;
}
constexpr int tw_stage_offset(int L, int NS) {
  int ns = 16, rem = L / 16, off = 0;
  while (ns < NS) {
    int R = rem >= 16 ? 16 : rem;
    off += R * ns;
    ns *= R;
    rem /= R;
  }
  return off;
}

template <int L, int R, int NS, bool FIRST, bool FIRST_SMEM, bool LAST, bool INV, class Lay>
__device__ __forceinline__ void ct_stage(cd (&v)[16], cd* sm, const cd* tws, int t, int line,
                                         const Lay& lay) {
  constexpr int T = L / 16, NB = 16 / R, LR = L / R;
  constexpr int OFF = FIRST ? 0 : tw_stage_offset(L, NS);
  cd a[16];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
    const int k = j & (NS - 1);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cd x;
      if (FIRST && !FIRST_SMEM) x = v[b * R + r];
      else x = ld_cd(sm + lay.at(line, j + r * LR));
      if (!FIRST && r > 0) {
        const cd w = tws[OFF + r * NS + k];
        x = INV ? cmul(x, w) : cmulc(x, w);
      }
      a[b * R + r] = x;
    }
    Dft<R, INV>::run(a + b * R);
  }
  if (!FIRST || FIRST_SMEM) __syncthreads();  // all reads done before in-place writes
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
    const int k = j & (NS - 1);
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (LAST) v[b + r * NB] = a[b * R + r];
      else st_cd(sm + lay.at(line, base + r * NS), a[b * R + r]);
    }
  }
  if (!LAST) __syncthreads();
}

template <int L, int NS, int REM, bool FIRST, bool FIRST_SMEM, bool INV, class Lay>
struct CtStages {
  static __device__ __forceinline__ void run(cd (&v)[16], cd* sm, const cd* tws, int t, int line,
                                             const Lay& lay) {
    constexpr int R = REM >= 16 ? 16 : REM;
    constexpr bool LAST = (REM == R);
    ct_stage<L, R, NS, FIRST, FIRST_SMEM, LAST, INV>(v, sm, tws, t, line, lay);
    if constexpr (!LAST)
      CtStages<L, NS * R, REM / R, false, false, INV, Lay>::run(v, sm, tws, t, line, lay);
  }
};

// Register contract as line_fft; L must be a power of two >= 16; tws is the
// stage-major table of L (tw_stage_size(L) entries).
template <int L, bool INV, bool FIRST_SMEM = false, class Lay>
__device__ __forceinline__ void line_fft_ct(cd (&v)[16], cd* sm, const cd* tws, int t, int line,
                                            const Lay& lay) {
  static_assert(L >= 16 && (L & (L - 1)) == 0, "compile-time FFT needs a power of two >= 16");
  CtStages<L, 1, L, true, FIRST_SMEM, INV, Lay>::run(v, sm, tws, t, line, lay);
}

// Twiddle table W_L^m = exp(+2 pi i m / L), m < L, into shared memory.
__device__ __forceinline__ void load_twiddles(cd* dst, const cd* src, int L) {
  for (int i = threadIdx.x; i < L; i += blockDim.x) dst[i] = ldg_cd(src + i);
}

// The same in two halves, so a kernel can issue the global loads before a
// dependent load chain (image state -> ring slot -> tile) and park them in
// shared memory after it: the first two entries per thread travel in registers.
struct TwiddleRegs {
  cd r[2];
};
__device__ __forceinline__ TwiddleRegs twiddles_issue(const cd* src, int L) {
  TwiddleRegs q;
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    q.r[j] = i < L ? ldg_cd(src + i) : cd{0.0, 0.0};
  }
  return q;
}
__device__ __forceinline__ void twiddles_park(cd* dst, const cd* src, int L, const TwiddleRegs& q) {
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int i = threadIdx.x + j * blockDim.x;
    if (i < L) dst[i] = q.r[j];
  }
  for (int i = threadIdx.x + 2 * blockDim.x; i < L; i += blockDim.x) dst[i] = ldg_cd(src + i);
}

}  // namespace redve
