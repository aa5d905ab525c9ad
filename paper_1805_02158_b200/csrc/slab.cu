// Primitives for the spatially partitioned solve (BASELINE.json configs[4]):
// every rank holds a row slab of one huge image (+ halos) and calls these on
// its slab; the partial sums they return are combined by an allreduce on the
// host side (torch.distributed / NCCL).  All reductions are deterministic:
// fixed-size per-CTA partials summed in CTA order.
#include "kernels.cuh"
#include "slab.cuh"

namespace redve {

static inline int nblocks(long long n) {
  long long b = (n + 255) / 256;
  return (int)(b > 296 ? 296 : (b < 1 ? 1 : b));
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

__global__ void k_vec_finish(const double* part, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nb; ++i) s += part[i];
    *out = s;
  }
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

// sum over the interior rows [h, h + rows) of ((H x)(u,v) - y_up(u,v))^2 at the
// GLOBAL measurement lattice ((row0 + u) mod Hg == 0 mod f, v == 0 mod f).
__global__ void k_fidelity(int Hext, int W, int row0, int Hg, int h, int rows, int f,
                           const double* taps, int k, const double* x, const double* yup,
                           double* part) {
  const int r = k / 2;
  double acc[1] = {0.0};
  const long long n = (long long)rows * W;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int u = h + (int)(idx / W), v = (int)(idx % W);
    const int g = (int)(((long long)row0 + u) % Hg);
    if ((g % f) || (v % f)) continue;
    double hx = 0.0;
    for (int a = 0; a < k; ++a)
      for (int c = 0; c < k; ++c)
        hx = fma(taps[a * k + c], x[(long long)wrap(u - (a - r), Hext) * W + wrap(v - (c - r), W)],
                 hx);
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
  const int nb = nblocks((long long)rows * W);
  k_fidelity<<<nb, 256, 0, s>>>(Hext, W, row0, Hg, h, rows, f, taps, k, x, yup, part);
  k_vec_finish<<<1, 32, 0, s>>>(part, nb, out);
}

// Gram of the differences of `rows` window vectors (row-major [rows][n]):
// G[i][j] = sum_p (w_{i+1} - w_i)(w_{j+1} - w_j), i, j < rows-1.  Per-CTA
// partials, summed in CTA order by k_gram_finish.
__global__ void k_window_gram(int rows, long long n, const double* w, double* part) {
  const int kp1 = rows - 1;
  const int ng = kp1 * (kp1 + 1) / 2;
  double acc[MAXKP1 * (MAXKP1 + 1) / 2];
  for (int i = 0; i < ng; ++i) acc[i] = 0.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    double d[MAXKP1];
    double prev = w[p];
    for (int j = 0; j < kp1; ++j) {
      const double nx = w[(long long)(j + 1) * n + p];
      d[j] = nx - prev;
      prev = nx;
    }
    int q = 0;
    for (int i = 0; i < kp1; ++i)
      for (int j = i; j < kp1; ++j) {
        acc[q] = fma(d[i], d[j], acc[q]);
        ++q;
      }
  }
  __shared__ double red[32];
  for (int i = 0; i < ng; ++i) {
    double one[1] = {acc[i]};
    block_sum<1>(one, red);
    if (threadIdx.x == 0) part[(long long)blockIdx.x * ng + i] = one[0];
  }
}
__global__ void k_gram_finish(const double* part, int nb, int kp1, double* G) {
  if (threadIdx.x || blockIdx.x) return;
  const int ng = kp1 * (kp1 + 1) / 2;
  int q = 0;
  for (int i = 0; i < kp1; ++i)
    for (int j = i; j < kp1; ++j) {
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s += part[(long long)b * ng + q];
      G[i * kp1 + j] = s;
      G[j * kp1 + i] = s;
      ++q;
    }
}
void launch_window_gram(int rows, long long n, const double* w, double* part, double* G,
                        cudaStream_t s) {
  const int nb = nblocks(n);
  k_window_gram<<<nb, 256, 0, s>>>(rows, n, w, part);
  k_gram_finish<<<1, 32, 0, s>>>(part, nb, rows - 1, G);
}

// out = w_0 + sum_{j<ke} xi_j (w_{j+1} - w_j)
__global__ void k_window_combine(long long n, const double* w, int ke, const double* xi,
                                 double* out) {
  __shared__ double s_xi[MAXKP1];
  if (threadIdx.x < ke) s_xi[threadIdx.x] = xi[threadIdx.x];
  __syncthreads();
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    double prev = w[p], acc = prev;
    for (int j = 0; j < ke; ++j) {
      const double nx = w[(long long)(j + 1) * n + p];
      acc = fma(s_xi[j], nx - prev, acc);
      prev = nx;
    }
    out[p] = acc;
  }
}
void launch_window_combine(long long n, const double* w, int ke, const double* xi, double* out,
                           cudaStream_t s) {
  k_window_combine<<<nblocks(n), 256, 0, s>>>(n, w, ke, xi, out);
}

}  // namespace redve
