// Shared helpers for the fused objective evaluation (cost.cu, fourier.cu).
#pragma once

#include "denoise.cuh"

namespace redve {

// Padded tile: element (i, c) at i*stride + c + c/16 -- conflict-free for the
// contiguous 16-column spans each thread reads.
struct TileLayout {
  int stride;
  __device__ __forceinline__ int at(int i, int c) const { return i * stride + c + (c >> 4); }
  static REDVE_HD int stride_for(int W) { return W + (W >> 4) + 1; }
};

// c within [-radius, W + radius): wrap with one compare (no integer division).
__device__ __forceinline__ int edge_wrap(int c, int W) {
  return c < 0 ? c + W : (c >= W ? c - W : c);
}

struct Sorted3 {
  cd lo, mid, hi;
};
__device__ __forceinline__ void sort2c(cd& a, cd& b) {
  sort2(a.x, b.x);
  sort2(a.y, b.y);
}
__device__ __forceinline__ Sorted3 sorted_col(cd a, cd b, cd c) {
  sort2c(a, b);
  sort2c(b, c);
  sort2c(a, b);
  return Sorted3{a, b, c};
}
__device__ __forceinline__ double med3d(double a, double b, double c) {
  return dmax(dmin(a, b), dmin(dmax(a, b), c));
}
// Median of the 3x3 block whose columns are A, B, C (each sorted): exact
// selection  med3( max(lows), med3(mids), min(highs) )  -- 2x fewer
// comparisons than the 19-comparator network when columns are shared.
__device__ __forceinline__ cd median_cols(const Sorted3& A, const Sorted3& B, const Sorted3& C) {
  cd r;
  r.x = med3d(dmax(dmax(A.lo.x, B.lo.x), C.lo.x), med3d(A.mid.x, B.mid.x, C.mid.x),
              dmin(dmin(A.hi.x, B.hi.x), C.hi.x));
  r.y = med3d(dmax(dmax(A.lo.y, B.lo.y), C.lo.y), med3d(A.mid.y, B.mid.y, C.mid.y),
              dmin(dmin(A.hi.y, B.hi.y), C.hi.y));
  return r;
}

// Medians of two neighbouring 3x3 windows, columns (A, B, C) and (B, C, D):
// max(B.lo, C.lo), min(B.hi, C.hi) and the ordered pair (B.mid, C.mid) are
// shared, 3 of the 9 min/max/compare-swaps per output pair (same values as two
// median_cols calls: every step selects one of its inputs).
__device__ __forceinline__ void median_pair1(double al, double am, double ah, double bl, double bm,
                                             double bh, double cl, double cm, double ch, double dl,
                                             double dm, double dh, double& o0, double& o1) {
  const double lbc = dmax(bl, cl), hbc = dmin(bh, ch);
  const double p = dmin(bm, cm), q = dmax(bm, cm);
  o0 = med3d(dmax(al, lbc), dmax(p, dmin(q, am)), dmin(ah, hbc));
  o1 = med3d(dmax(lbc, dl), dmax(p, dmin(q, dm)), dmin(hbc, dh));
}

__device__ __forceinline__ void median_pair(const Sorted3& A, const Sorted3& B, const Sorted3& C,
                                            const Sorted3& D, cd& r0, cd& r1) {
  median_pair1(A.lo.x, A.mid.x, A.hi.x, B.lo.x, B.mid.x, B.hi.x, C.lo.x, C.mid.x, C.hi.x, D.lo.x,
               D.mid.x, D.hi.x, r0.x, r1.x);
  median_pair1(A.lo.y, A.mid.y, A.hi.y, B.lo.y, B.mid.y, B.hi.y, C.lo.y, C.mid.y, C.hi.y, D.lo.y,
               D.mid.y, D.hi.y, r0.y, r1.y);
}

// k x k periodic convolution over the 16 contiguous columns [c0, c0+16) of
// tile row ti (pairs), K known at compile time.  Same terms and per-output
// order (ta outer, tb inner) as the runtime loop below.
template <int K, class Wrap>
__device__ __forceinline__ void conv_span(cd (&f)[16], const cd* tile, const TileLayout& tl, int ti,
                                          int c0, const double* taps, Wrap wrapc) {
  constexpr int r = K / 2;
#pragma unroll
  for (int j = 0; j < 16; ++j) f[j] = cd{0.0, 0.0};
  // the tap rows stay a loop: fully unrolled, the 5x5 body is ~800 FMAs of
  // straight-line code per span and a single-image solve (configs[0], few
  // warps per SM) stalls on instruction fetch (ncu: no_instruction)
#pragma unroll 1
  for (int ta = 0; ta < K; ++ta) {
    cd row[16 + K - 1];  // columns c0 - r .. c0 + 15 + r of tile row ti - (ta - r)
#pragma unroll
    for (int u = 0; u < 16 + K - 1; ++u) row[u] = ld_cd(tile + tl.at(ti - (ta - r), wrapc(c0 - r + u)));
#pragma unroll
    for (int tb = 0; tb < K; ++tb) {
      const double w = taps[ta * K + tb];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const cd xx = row[j + K - 1 - tb];  // column c0 + j - (tb - r)
        f[j].x = fma(w, xx.x, f[j].x);
        f[j].y = fma(w, xx.y, f[j].y);
      }
    }
  }
}

// f over the 16 contiguous columns [c0, c0+16) of tile row ti (pairs).
// WRAP(c) maps a column in [-r, W + r) into [0, W).
template <int DK, class Wrap>
__device__ __forceinline__ void denoise_span(cd (&f)[16], const cd* tile, const TileLayout& tl,
                                             int ti, int c0, int ksize, const double* taps,
                                             Wrap wrapc) {
  if (DK == DN_MEDIAN3) {
    auto col = [&](int j) {
      const int c = wrapc(c0 + j);
      return sorted_col(ld_cd(tile + tl.at(ti - 1, c)), ld_cd(tile + tl.at(ti, c)),
                        ld_cd(tile + tl.at(ti + 1, c)));
    };
    Sorted3 A = col(-1), B = col(0);
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
      Sorted3 C = col(j + 1), D = col(j + 2);
      median_pair(A, B, C, D, f[j], f[j + 1]);
      A = C;
      B = D;
    }
  } else if (DK == DN_CONV && (ksize == 3 || ksize == 5)) {
    // compile-time taps loop: the 16 accumulator chains interleave
    if (ksize == 3) conv_span<3>(f, tile, tl, ti, c0, taps, wrapc);
    else conv_span<5>(f, tile, tl, ti, c0, taps, wrapc);
  } else if (DK == DN_CONV) {
    const int r = ksize >> 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      cd acc = cd{0.0, 0.0};
      for (int ta = 0; ta < ksize; ++ta) {
        for (int tb = 0; tb < ksize; ++tb) {
          const double w = taps[ta * ksize + tb];
          const cd xx = ld_cd(tile + tl.at(ti - (ta - r), wrapc(c0 + j - (tb - r))));
          acc.x = fma(w, xx.x, acc.x);
          acc.y = fma(w, xx.y, acc.y);
        }
      }
      f[j] = acc;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) f[j] = ld_cd(tile + tl.at(ti, wrapc(c0 + j)));
  }
}

// K x K correlation at the pixel pair (i, j), (i, j+1), K known at compile
// time: the K+1 wrapped columns are formed once and every row's K+1 values
// feed both outputs (same terms and order as fk_pair's runtime loop).
template <int K>
__device__ __forceinline__ void conv_pair(const double* x, int H, int W, int i, int j,
                                          const double* taps, double& f0, double& f1) {
  constexpr int r = K / 2;
  int cols[K + 1];  // columns j - r .. j + 1 + r
#pragma unroll
  for (int u = 0; u <= K; ++u) cols[u] = wrap_fast(j - r + u, W);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll
  for (int ta = 0; ta < K; ++ta) {
    const double* row = x + (long long)wrap_fast(i - (ta - r), H) * W;
    double v[K + 1];
#pragma unroll
    for (int u = 0; u <= K; ++u) v[u] = __ldg(row + cols[u]);
#pragma unroll
    for (int tb = 0; tb < K; ++tb) {
      const double w = taps[ta * K + tb];
      a0 = fma(w, v[2 * r - tb], a0);
      a1 = fma(w, v[2 * r - tb + 1], a1);
    }
  }
  f0 = a0;
  f1 = a1;
}

// f(x) at the pixel pair (i, j), (i, j+1) of one image from L1-resident
// neighbours (periodic): the streaming kernels' denoiser (cost.cu k_cost_fp,
// kernels.cu k_median3_pairs).
template <int DK>
__device__ __forceinline__ void fk_pair(const double* x, int H, int W, int i, int j,
                                        const DenoiseArgs& dn, const double* taps,
                                        double& f0, double& f1) {
  if (DK == DN_MEDIAN3) {
    const int im = wrap_fast(i - 1, H), ip = wrap_fast(i + 1, H);
    const int jm = edge_wrap(j - 1, W), jp = edge_wrap(j + 2, W);
    const double* r0 = x + (long long)im * W;
    const double* r1 = x + (long long)i * W;
    const double* r2 = x + (long long)ip * W;
    double c[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int cq = q == 0 ? jm : (q == 3 ? jp : j + q - 1);
      double a = __ldg(r0 + cq), b = __ldg(r1 + cq), e = __ldg(r2 + cq);
      sort2(a, b);
      sort2(b, e);
      sort2(a, b);
      c[q][0] = a;
      c[q][1] = b;
      c[q][2] = e;
    }
    median_pair1(c[0][0], c[0][1], c[0][2], c[1][0], c[1][1], c[1][2], c[2][0], c[2][1], c[2][2],
                 c[3][0], c[3][1], c[3][2], f0, f1);
  } else if (DK == DN_CONV && (dn.ksize == 3 || dn.ksize == 5)) {
    if (dn.ksize == 5) conv_pair<5>(x, H, W, i, j, taps, f0, f1);
    else conv_pair<3>(x, H, W, i, j, taps, f0, f1);
  } else if (DK == DN_CONV) {
    const int k = dn.ksize, r = k >> 1;
    double a0 = 0.0, a1 = 0.0;
    for (int ta = 0; ta < k; ++ta) {
      const double* row = x + (long long)wrap_fast(i - (ta - r), H) * W;
      for (int tb = 0; tb < k; ++tb) {
        const double w = taps[ta * k + tb];
        a0 = fma(w, __ldg(row + wrap_fast(j - (tb - r), W)), a0);
        a1 = fma(w, __ldg(row + wrap_fast(j + 1 - (tb - r), W)), a1);
      }
    }
    f0 = a0;
    f1 = a1;
  } else {
    const double2 v = __ldg(reinterpret_cast<const double2*>(x + (long long)i * W + j));
    f0 = v.x;
    f1 = v.y;
  }
}

// Periodic k x k correlation (corr) or convolution at the pixel pair
// (i, j), (i, j+1): out = sum_ab taps[a][b] x(i +- (a-r), j +- (b-r)).
__device__ __forceinline__ void stencil_pair(const double* x, int H, int W, int i, int j,
                                             const double* taps, int k, int corr,
                                             double& f0, double& f1) {
  const int r = k >> 1;
  double a0 = 0.0, a1 = 0.0;
  for (int ta = 0; ta < k; ++ta) {
    const int da = corr ? (ta - r) : (r - ta);
    const double* row = x + (long long)wrap_fast(i + da, H) * W;
    for (int tb = 0; tb < k; ++tb) {
      const int db = corr ? (tb - r) : (r - tb);
      const double w = taps[ta * k + tb];
      a0 = fma(w, __ldg(row + wrap_fast(j + db, W)), a0);
      a1 = fma(w, __ldg(row + wrap_fast(j + 1 + db, W)), a1);
    }
  }
  f0 = a0;
  f1 = a1;
}

}  // namespace redve
