// Denoiser stencils evaluated from a shared-memory tile (denoisers.py:21-46 +
// the BASELINE.json 3x3 median).  The tile holds two images of a batch pair
// interleaved as one complex value (re = image 2p, im = image 2p+1), so one
// 16-byte shared load feeds both images.
#pragma once

#include "common.cuh"

namespace redve {

enum DenoiseKind : int {
  DN_IDENTITY = 0,   // f(x) = x                                (denoisers.py:21-27)
  DN_CONV = 1,       // circular convolution with k x k taps    (denoisers.py:30-46)
  DN_MEDIAN3 = 2,    // periodic 3x3 median (bit-exact order statistic)
  DN_EXTERNAL = 3,   // f precomputed into a buffer (filter bank, patch-weighted, host plug-in)
};

struct DenoiseArgs {
  int kind;
  int ksize;          // DN_CONV taps size (odd)
  int radius;         // halo rows/cols the stencil needs
  const double* taps; // device, ksize*ksize, row-major taps[a][b]
};

// One comparison, two selects (fmin/fmax cost two compares plus NaN fix-ups on
// sm_100; iterates reaching a denoiser are finite, so plain ordering is exact).
__device__ __forceinline__ void sort2(double& a, double& b) {
  const bool sw = b < a;
  const double lo = sw ? b : a, hi = sw ? a : b;
  a = lo;
  b = hi;
}
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }

// Median of 9 with the 19-comparator network (exact selection).
__device__ __forceinline__ double median9(double* p) {
  sort2(p[1], p[2]); sort2(p[4], p[5]); sort2(p[7], p[8]);
  sort2(p[0], p[1]); sort2(p[3], p[4]); sort2(p[6], p[7]);
  sort2(p[1], p[2]); sort2(p[4], p[5]); sort2(p[7], p[8]);
  sort2(p[0], p[3]); sort2(p[5], p[8]); sort2(p[4], p[7]);
  sort2(p[3], p[6]); sort2(p[1], p[4]); sort2(p[2], p[5]);
  sort2(p[4], p[7]); sort2(p[4], p[2]); sort2(p[6], p[4]);
  sort2(p[4], p[2]);
  return p[4];
}

__device__ __forceinline__ int wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}
// periodic index, cheap when already in range (tile halos mostly are)
__device__ __forceinline__ int wrap_fast(int i, int n) {
  return ((unsigned)i < (unsigned)n) ? i : wrap(i, n);
}

// f at (tile row ti, column c) for both images of the pair.  `tile` is
// [rows][W] complex; `taps` in shared memory.
__device__ __forceinline__ cd denoise_at(const cd* tile, int W, int ti, int c, int kind, int ksize,
                                         const double* taps) {
  if (kind == DN_MEDIAN3) {
    double re[9], im[9];
    int q = 0;
#pragma unroll
    for (int a = -1; a <= 1; ++a) {
#pragma unroll
      for (int b = -1; b <= 1; ++b) {
        cd v = ld_cd(tile + (ti + a) * W + wrap(c + b, W));
        re[q] = v.x;
        im[q] = v.y;
        ++q;
      }
    }
    return cd{median9(re), median9(im)};
  }
  if (kind == DN_CONV) {
    const int r = ksize >> 1;
    cd acc = cd{0.0, 0.0};
    // f[i,j] = sum_{a,b} taps[a][b] * x[i-(a-r), j-(b-r)]   (convolution)
    for (int a = 0; a < ksize; ++a) {
      const cd* row = tile + (ti - (a - r)) * W;
      for (int b = 0; b < ksize; ++b) {
        const double w = taps[a * ksize + b];
        cd v = ld_cd(row + wrap(c - (b - r), W));
        acc.x = fma(w, v.x, acc.x);
        acc.y = fma(w, v.y, acc.y);
      }
    }
    return acc;
  }
  return ld_cd(tile + ti * W + c);  // identity / external
}

}  // namespace redve
