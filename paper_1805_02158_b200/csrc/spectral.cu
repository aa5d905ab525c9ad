// Spectral route kernels (see spectral.cuh): the fixed-point step, the cost
// cadence and the DFT staging of the Fourier-domain iteration for linear
// shift-invariant denoisers.
#include "spectral.cuh"

namespace redve {

namespace {

constexpr int SP_THREADS = 256;

inline int cdivs(long long a, long long b) { return (int)((a + b - 1) / b); }

// cost_finish (kernels.cuh) reads these fields only
__device__ __forceinline__ CostArgs cost_view(int H, int W, int mode, double sigma, double alpha,
                                              const StepCtl& ctl, const TraceBufs& tr) {
  CostArgs c;
  c.H = H;
  c.W = W;
  c.mode = mode;
  c.sigma = sigma;
  c.alpha = alpha;
  c.ctl = ctl;
  c.tr = tr;
  return c;
}

// (1/N)-scaled data / prior / reference sums of spectrum X at frequency i
__device__ __forceinline__ void cost_terms(const SpecConsts& k, int b, long long N, long long i,
                                           cd x, double& fid, double& reg, double& ssd) {
  const cd h = ldg_cd(k.hh + i);
  const cd y = ldg_cd(k.yh + (long long)b * N + i);
  const cd r = cd{fma(h.x, x.x, -fma(h.y, x.y, y.x)), fma(h.x, x.y, fma(h.y, x.x, -y.y))};
  fid = fma(r.x, r.x, fma(r.y, r.y, fid));
  reg = fma(fma(x.x, x.x, x.y * x.y), __ldg(k.wr + i), reg);
  if (k.rh) {
    const cd q = ldg_cd(k.rh + (long long)b * N + i);
    const double dx = x.x - q.x, dy = x.y - q.y;
    ssd = fma(dx, dx, fma(dy, dy, ssd));
  }
}

}  // namespace

int spec_chunks(int B, long long N) {
  // small batches are latency bound: one frequency per thread, as many CTAs as
  // that takes (up to ~8 per SM); large batches: ~8 resident CTAs per SM overall
  int c = cdivs(148LL * 8, B);
  const int cmax = cdivs(N, SP_THREADS);
  if (c > cmax) c = cmax;
  return c < 1 ? 1 : c;
}

// X+ = Xb + m X; step-norm sums; on cadence the cost / PSNR of X+ as well.
__global__ void __launch_bounds__(SP_THREADS) k_spec_step(SpecStepArgs a) {
  const int b = blockIdx.y;
  ImgState& st = a.st[b];
  if (!takes_step(st, a.ctl.phase)) return;
  const long long N = (long long)a.H * a.W;
  const cd* x = reinterpret_cast<const cd*>(a.cur.at(b, a.st));
  cd* xn = reinterpret_cast<cd*>(a.nxt.at(b, a.st));
  const cd* xb = a.k.xb + (long long)b * N;
  double acc[6] = {0, 0, 0, 0, 0, 0};  // d2, x2, nonfinite, fid, reg, ssd
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    const cd v = ld_cd(x + i), m = ldg_cd(a.k.m + i), c = ldg_cd(xb + i);
    const cd u = cd{fma(m.x, v.x, fma(-m.y, v.y, c.x)), fma(m.x, v.y, fma(m.y, v.x, c.y))};
    st_cd(xn + i, u);
    const double dx = u.x - v.x, dy = u.y - v.y;
    acc[0] = fma(dx, dx, fma(dy, dy, acc[0]));
    acc[1] = fma(v.x, v.x, fma(v.y, v.y, acc[1]));
    acc[2] += (isfinite(u.x) && isfinite(u.y)) ? 0.0 : 1.0;
    if (a.cadence) cost_terms(a.k, b, N, i, u, acc[3], acc[4], acc[5]);
  }
  __shared__ double red[32 * 6];
  block_sum<6>(acc, red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0)
    for (int q = 0; q < 6; ++q) a.partials[((long long)b * nblk + blockIdx.x) * 6 + q] = acc[q];
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double t[6];
  if (lastb) gather_partials<6>(a.partials + (long long)b * nblk * 6, nblk, t, red);
  if (lastb && threadIdx.x == 0) {
    StepCtl c = a.ctl;
    c.defer_commit = a.cadence;
    record_step(st, b, t[0], t[1], t[2], a.S, c, a.tr);
    if (a.cadence) {
      if (st.k % c.log_every == 0) {
        const double inv = 1.0 / (double)N;
        const CostArgs ca = cost_view(a.H, a.W, COST_RECORD, a.sigma, a.alpha, c, a.tr);
        cost_finish(st, b, t[3] * inv, t[4] * inv, t[5] * inv, a.k.rh != nullptr, ca);
      }
      commit_step(st, c.phase);
    }
  }
}

// note_initial / finalize costs of the current spectrum (solvers.py:219-223, 255-262)
__global__ void __launch_bounds__(SP_THREADS) k_spec_cost(SpecCostArgs a) {
  const int b = blockIdx.y;
  ImgState& st = a.st[b];
  if (a.mode == COST_FINAL && st.err != ERR_NONE) return;
  const long long N = (long long)a.H * a.W;
  const cd* x = reinterpret_cast<const cd*>(a.x.at(b, a.st));
  double acc[3] = {0, 0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    cost_terms(a.k, b, N, i, ld_cd(x + i), acc[0], acc[1], acc[2]);
  __shared__ double red[32 * 3];
  block_sum<3>(acc, red);
  const int nblk = gridDim.x;
  if (threadIdx.x == 0)
    for (int q = 0; q < 3; ++q) a.partials[((long long)b * nblk + blockIdx.x) * 3 + q] = acc[q];
  __shared__ int s_last;
  const bool lastb = last_block_of_group(a.counters + b, nblk, &s_last);
  double t[3];
  if (lastb) gather_partials<3>(a.partials + (long long)b * nblk * 3, nblk, t, red);
  if (lastb && threadIdx.x == 0) {
    const double inv = 1.0 / (double)N;
    const CostArgs ca = cost_view(a.H, a.W, a.mode, a.sigma, a.alpha, a.ctl, a.tr);
    cost_finish(st, b, t[0] * inv, t[1] * inv, t[2] * inv, a.k.rh != nullptr, ca);
  }
}

__global__ void k_spec_pack(const double* x, long long N, cd* out, long long odist, int* bad) {
  const int b = blockIdx.y;
  int nf = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    const double v = x[(long long)b * N + i];
    nf |= !isfinite(v);
    st_cd(out + (long long)b * odist + i, cd{v, 0.0});
  }
  if (bad && __syncthreads_or(nf) && threadIdx.x == 0) atomicOr(bad, 1);
}

__global__ void k_spec_embed(const double* taps, int k, int H, int W, cd* out) {
  const long long N = (long long)H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    st_cd(out + i, cd{0.0, 0.0});
  __syncthreads();  // single CTA: zero fill before the taps land
  const int r = k / 2;
  for (int t = threadIdx.x; t < k * k; t += blockDim.x) {
    const int ta = t / k, tb = t - ta * k;
    int i = (ta - r) % H, j = (tb - r) % W;
    i += i < 0 ? H : 0;
    j += j < 0 ? W : 0;
    // taps overlapping after wrap (k > side) accumulate, as the embedding's roll does
    atomicAdd(&reinterpret_cast<double*>(out + (long long)i * W + j)[0], taps[t]);
  }
}

__global__ void k_spec_consts(const cd* hf, const double* g, double alpha, long long N, cd* m,
                              double* wr) {
  const double scale = (double)N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x) {
    const cd h = hf ? ld_cd(hf + i) : cd{1.0, 0.0};
    const double invd = g[i] * scale;  // g = 1 / (d H W)
    st_cd(m + i, cd{alpha * h.x * invd, alpha * h.y * invd});
    wr[i] = 1.0 - h.x;
  }
}

__global__ void k_spec_pick(cd* out, View cur, const double* best, long long N,
                            const ImgState* st) {
  const int b = blockIdx.y;
  const cd* src = reinterpret_cast<const cd*>(st[b].use_best ? best + (long long)b * 2 * N
                                                             : cur.at(b, st));
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    st_cd(out + (long long)b * N + i, ld_cd(src + i));
}

__global__ void k_spec_real(const cd* z, double* out, long long N, double scale) {
  const int b = blockIdx.y;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
       i += (long long)gridDim.x * blockDim.x)
    out[(long long)b * N + i] = z[(long long)b * N + i].x * scale;
}

void launch_spec_step(const SpecStepArgs& a, cudaStream_t s) {
  k_spec_step<<<dim3(spec_chunks(a.B, (long long)a.H * a.W), a.B), SP_THREADS, 0, s>>>(a);
}
void launch_spec_cost(const SpecCostArgs& a, cudaStream_t s) {
  k_spec_cost<<<dim3(spec_chunks(a.B, (long long)a.H * a.W), a.B), SP_THREADS, 0, s>>>(a);
}
void launch_spec_pack(const double* x, int B, long long N, cd* out, long long odist, int* bad,
                      cudaStream_t s) {
  k_spec_pack<<<dim3(spec_chunks(B, N), B), SP_THREADS, 0, s>>>(x, N, out, odist, bad);
}
void launch_spec_embed(const double* taps, int k, int H, int W, cd* out, cudaStream_t s) {
  k_spec_embed<<<1, 1024, 0, s>>>(taps, k, H, W, out);
}
void launch_spec_consts(const cd* hf, const double* g, double alpha, long long N, cd* m,
                        double* wr, cudaStream_t s) {
  k_spec_consts<<<cdivs(N, SP_THREADS * 4), SP_THREADS, 0, s>>>(hf, g, alpha, N, m, wr);
}
void launch_spec_pick(cd* out, View cur, const double* best, int B, long long N,
                      const ImgState* st, cudaStream_t s) {
  k_spec_pick<<<dim3(spec_chunks(B, N), B), SP_THREADS, 0, s>>>(out, cur, best, N, st);
}
void launch_spec_real(const cd* z, double* out, int B, long long N, double scale, cudaStream_t s) {
  k_spec_real<<<dim3(spec_chunks(B, N), B), SP_THREADS, 0, s>>>(z, out, N, scale);
}

}  // namespace redve
