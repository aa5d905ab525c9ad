// Primitives for the spatially partitioned solve (BASELINE.json configs[4]):
// every rank holds a row slab of one huge image (+ halos) and calls these on
// its slab; the partial sums they return are combined by an allreduce on the
// host side (torch.distributed / NCCL).  All reductions are deterministic:
// fixed-size per-CTA partials summed in CTA order.
#include "kernels.cuh"
#include "slab.cuh"

namespace redve {

// enough 256-thread CTAs for 8 per SM (4 for the Gram), fewer for small vectors
static inline int nblocks(long long n, int cap = SLAB_BLOCKS) {
  long long b = (n + 255) / 256;
  return (int)(b > cap ? cap : (b < 1 ? 1 : b));
}

// out[k] (per CTA) for k in [0, K): sums of x*y (DOT), (x-y)^2 (DIST2)
template <int OP>
__global__ void k_vec_reduce(long long n, const double* x, const double* y, double* part) {
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double a = x[i], b = y[i];
    if (OP == 0) acc[0] = fma(a, b, acc[0]);
    else {
      const double d = a - b;
      acc[0] = fma(d, d, acc[0]);
    }
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}

// one warp: lane-strided sums, then a fixed shuffle tree (deterministic)
__global__ void k_vec_finish(const double* part, int nb, double* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32) s += part[i];
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (threadIdx.x == 0) *out = s;
}

void launch_vec_reduce(int op, long long n, const double* x, const double* y, double* part,
                       double* out, cudaStream_t s) {
  const int nb = nblocks(n);
  if (op == 0) k_vec_reduce<0><<<nb, 256, 0, s>>>(n, x, y, part);
  else k_vec_reduce<1><<<nb, 256, 0, s>>>(n, x, y, part);
  k_vec_finish<<<1, 32, 0, s>>>(part, nb, out);
}

// y = a*x + b*y
__global__ void k_vec_axpby(long long n, double a, const double* x, double b, double* y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}
void launch_vec_axpby(long long n, double a, const double* x, double b, double* y,
                      cudaStream_t s) {
  k_vec_axpby<<<nblocks(n), 256, 0, s>>>(n, a, x, b, y);
}

// Halo push over peer memory: the slab x [rows][W] goes into the interior of
// this rank's extended buffer, and in the same pass its first `halo` rows are
// stored into the previous rank's bottom halo and its last `halo` rows into
// the next rank's top halo (pointers opened over CUDA IPC, or into this
// rank's own buffer for a single-rank periodic wrap).  16-byte accesses when
// every row start is 16-byte aligned.
template <typename V>
__global__ void k_halo_push(long long rows, long long Wv, long long halo, const V* x, V* ext,
                            V* prev_bot, V* next_top) {
  const long long n = rows * Wv;
  const long long lo = halo * Wv, hi = (rows - halo) * Wv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const V v = x[i];
    ext[lo + i] = v;
    if (i < lo) prev_bot[i] = v;
    if (i >= hi) next_top[i - hi] = v;
  }
}
void launch_halo_push(int rows, int W, int halo, const double* x, double* ext, double* prev_bot,
                      double* next_top, cudaStream_t s) {
  const bool v2 = (W % 2 == 0) && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(ext) |
                                    reinterpret_cast<uintptr_t>(prev_bot) |
                                    reinterpret_cast<uintptr_t>(next_top)) % 16 == 0);
  if (v2) {
    const long long Wv = W / 2;
    k_halo_push<double2><<<nblocks((long long)rows * Wv), 256, 0, s>>>(
        rows, Wv, halo, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(ext),
        reinterpret_cast<double2*>(prev_bot), reinterpret_cast<double2*>(next_top));
  } else {
    k_halo_push<double><<<nblocks((long long)rows * W), 256, 0, s>>>(rows, W, halo, x, ext,
                                                                    prev_bot, next_top);
  }
}

// sum over the interior rows [h, h + rows) of ((H x)(u,v) - y_up(u,v))^2 at the
// GLOBAL measurement lattice ((row0 + u) mod Hg == 0 mod f, v == 0 mod f).
__global__ void k_fidelity(int Hext, int W, int row0, int Hg, int h, int rows, int f,
                           const double* taps, int k, const double* x, const double* yup,
                           double* part) {
  const int r = k / 2;
  double acc[1] = {0.0};
  // work items: (interior row, lattice column); rows off the lattice drop out a
  // warp at a time (the lattice test is per row, the columns are all on it)
  const int ncl = (W + f - 1) / f;
  const long long n = (long long)rows * ncl;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int u = h + (int)(idx / ncl), v = f * (int)(idx % ncl);
    const int g = (int)(((long long)row0 + u) % Hg);
    if (g % f) continue;
    double hx = 0.0;
    for (int a = 0; a < k; ++a) {
      int ua = u - (a - r);  // within one period of [0, Hext)
      ua = ua < 0 ? ua + Hext : (ua >= Hext ? ua - Hext : ua);
      const double* xr = x + (long long)ua * W;
      for (int c = 0; c < k; ++c) {
        int vc = v - (c - r);
        vc = vc < 0 ? vc + W : (vc >= W ? vc - W : vc);
        hx = fma(taps[a * k + c], xr[vc], hx);
      }
    }
    const double d = hx - yup[(long long)u * W + v];
    acc[0] = fma(d, d, acc[0]);
  }
  __shared__ double red[32];
  block_sum<1>(acc, red);
  if (threadIdx.x == 0) part[blockIdx.x] = acc[0];
}
void launch_fidelity(int Hext, int W, int row0, int Hg, int h, int rows, int f,
                     const double* taps, int k, const double* x, const double* yup, double* part,
                     double* out, cudaStream_t s) {
  const int nb = nblocks((long long)rows * ((W + f - 1) / f));
  k_fidelity<<<nb, 256, 0, s>>>(Hext, W, row0, Hg, h, rows, f, taps, k, x, yup, part);
  k_vec_finish<<<1, 32, 0, s>>>(part, nb, out);
}

// Gram of the differences of KP1+1 window vectors (row-major [KP1+1][n]):
// G[i][j] = sum_p (w_{i+1} - w_i)(w_{j+1} - w_j).  Per-CTA partials (upper
// triangle, row-major), summed in CTA order by k_gram_finish.
template <int KP1>
__global__ void __launch_bounds__(256) k_window_gram(long long n, const double* w, double* part) {
  constexpr int NG = KP1 * (KP1 + 1) / 2;
  double acc[NG];
#pragma unroll
  for (int i = 0; i < NG; ++i) acc[i] = 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    double v[KP1 + 1];
#pragma unroll
    for (int j = 0; j <= KP1; ++j) v[j] = w[(long long)j * n + p];
    double d[KP1];
#pragma unroll
    for (int j = 0; j < KP1; ++j) d[j] = v[j + 1] - v[j];
    int q = 0;
#pragma unroll
    for (int i = 0; i < KP1; ++i)
#pragma unroll
      for (int j = i; j < KP1; ++j) {
        acc[q] = fma(d[i], d[j], acc[q]);
        ++q;
      }
  }
  __shared__ double red[32];
#pragma unroll
  for (int i = 0; i < NG; ++i) {
    double one[1] = {acc[i]};
    block_sum<1>(one, red);
    if (threadIdx.x == 0) part[(long long)blockIdx.x * NG + i] = one[0];
  }
}
// one warp per Gram entry: lane-strided sums over the CTAs, fixed shuffle tree
__global__ void k_gram_finish(const double* part, int nb, int kp1, double* G) {
  const int ng = kp1 * (kp1 + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = warp; q < ng; q += blockDim.x >> 5) {
    double s = 0.0;
    for (int b = lane; b < nb; b += 32) s += part[(long long)b * ng + q];
    for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) {
      int i = 0, base = 0;
      while (q >= base + (kp1 - i)) {
        base += kp1 - i;
        ++i;
      }
      const int j = i + (q - base);
      G[i * kp1 + j] = s;
      G[j * kp1 + i] = s;
    }
  }
}
void launch_window_gram(int rows, long long n, const double* w, double* part, double* G,
                        cudaStream_t s) {
  const int nb = nblocks(n, GRAM_BLOCKS);
  switch (rows - 1) {
#define GRAM_CASE(K) \
  case K: k_window_gram<K><<<nb, 256, 0, s>>>(n, w, part); break;
    GRAM_CASE(1) GRAM_CASE(2) GRAM_CASE(3) GRAM_CASE(4) GRAM_CASE(5) GRAM_CASE(6)
    GRAM_CASE(7) GRAM_CASE(8) GRAM_CASE(9) GRAM_CASE(10) GRAM_CASE(11) GRAM_CASE(12)
#undef GRAM_CASE
    default: return;
  }
  k_gram_finish<<<1, 256, 0, s>>>(part, nb, rows - 1, G);
}

// out = w_0 + sum_{j<KE} xi_j (w_{j+1} - w_j)
template <int KE>
__global__ void __launch_bounds__(256) k_window_combine(long long n, const double* w,
                                                        const double* xi, double* out) {
  double c[KE];
#pragma unroll
  for (int j = 0; j < KE; ++j) c[j] = xi[j];
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    double v[KE + 1];
#pragma unroll
    for (int j = 0; j <= KE; ++j) v[j] = w[(long long)j * n + p];
    double acc = v[0];
#pragma unroll
    for (int j = 0; j < KE; ++j) acc = fma(c[j], v[j + 1] - v[j], acc);
    out[p] = acc;
  }
}
void launch_window_combine(long long n, const double* w, int ke, const double* xi, double* out,
                           cudaStream_t s) {
  const int nb = nblocks(n);
  switch (ke) {
#define COMB_CASE(K) \
  case K: k_window_combine<K><<<nb, 256, 0, s>>>(n, w, xi, out); break;
    COMB_CASE(1) COMB_CASE(2) COMB_CASE(3) COMB_CASE(4) COMB_CASE(5) COMB_CASE(6)
    COMB_CASE(7) COMB_CASE(8) COMB_CASE(9) COMB_CASE(10) COMB_CASE(11)
#undef COMB_CASE
    default: return;
  }
}

}  // namespace redve
