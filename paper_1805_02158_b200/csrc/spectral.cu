// Spectral route kernels (see spectral.cuh): the fixed-point step, the cost
// cadence and the DFT staging of the Fourier-domain iteration for linear
// shift-invariant denoisers.
#include <cooperative_groups.h>
#include <cstdlib>

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

// Several spectral steps in one launch: one cluster of SPC_CL CTAs per image
// holds the image's spectrum and its step constants (m, Xb) in shared memory,
// so a step costs no launch and no HBM round trip -- the new spectrum still
// lands in the ring (the VE window reads it).  Each step is k_spec_step's
// arithmetic verbatim (iterates bit-identical).  Its sums travel by DSMEM
// push: every CTA st.async's its 6 partial sums into every CTA's gather slot,
// completing on the receiver's mbarrier (no cluster-wide barrier, hence no
// release fence waiting on the ring stores); every CTA then sums the partials
// in the same fixed order and applies the record / cadence cost / commit to
// its own shared copy of the image state -- identical in every CTA; rank 0
// alone writes the traces and, at the end, the state.  A cadence step's
// best-iterate copy (k_copy_view) is done per CTA for its own frequencies.
// Small batches only (the launch-bound configs[0] regime).
constexpr int SPC_CL = 16, SPC_THREADS = 512, SPC_MAXF = 4096;  // frequencies per CTA

__device__ __forceinline__ unsigned spc_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned spc_mapa(unsigned addr, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__global__ void __launch_bounds__(SPC_THREADS) k_spec_steps(SpecStepArgs a, int nsteps,
                                                            unsigned cadence_mask, int copy_best,
                                                            double* best) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int b = blockIdx.y;
  const int rank = (int)cluster.block_rank();
  const long long N = (long long)a.H * a.W;
  const long long per = (N + SPC_CL - 1) / SPC_CL;
  const long long lo = rank * per, hi = lo + per < N ? lo + per : N;
  const int nf = (int)(hi > lo ? hi - lo : 0);
  extern __shared__ __align__(16) unsigned char spc_smem[];
  cd* xs = reinterpret_cast<cd*>(spc_smem);
  cd* ms = xs + SPC_MAXF;
  cd* bs = ms + SPC_MAXF;
  __shared__ double red[32 * 6];
  __shared__ __align__(16) double mine[6];
  __shared__ __align__(16) double gat[2][SPC_CL][6];  // by step parity, by sender rank
  __shared__ __align__(8) unsigned long long gbar[2];
  __shared__ ImgState sst;  // this CTA's copy of the image state
  __shared__ int s_go, s_copy;
  if (threadIdx.x == 0) {
    sst = a.st[b];
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(spc_smem_u32(&gbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  TraceBufs tr = a.tr;
  if (rank != 0) tr.cap = 0;  // shadow records: state only, no trace writes
  {  // the current spectrum and the step constants of my frequencies
    const cd* x = reinterpret_cast<const cd*>(a.cur.at(b, a.st)) + lo;
    const cd* xb = a.k.xb + (long long)b * N + lo;
    for (int j = threadIdx.x; j < nf; j += blockDim.x) {
      xs[j] = ld_cd(x + j);
      ms[j] = ldg_cd(a.k.m + lo + j);
      bs[j] = ldg_cd(xb + j);
    }
  }
  cluster.sync();  // every CTA's mbarriers are initialised before any push
  if (threadIdx.x == 0) s_go = takes_step(sst, a.ctl.phase);
  __syncthreads();
  for (int step = 0; step < nsteps && s_go; ++step) {
    const int buf = step & 1;
    const bool cadence = (cadence_mask >> step) & 1u;
    if (threadIdx.x == 0)  // this step's 16 partials (48 bytes each) complete the phase
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                       spc_smem_u32(&gbar[buf])),
                   "r"(SPC_CL * 48)
                   : "memory");
    cd* xn = reinterpret_cast<cd*>(a.nxt.at_state(b, sst)) + lo;
    double acc[6] = {0, 0, 0, 0, 0, 0};  // d2, x2, nonfinite, fid, reg, ssd
    for (int j = threadIdx.x; j < nf; j += blockDim.x) {
      const cd v = xs[j], m = ms[j], c = bs[j];
      const cd u = cd{fma(m.x, v.x, fma(-m.y, v.y, c.x)), fma(m.x, v.y, fma(m.y, v.x, c.y))};
      st_cd(xn + j, u);
      xs[j] = u;
      const double dx = u.x - v.x, dy = u.y - v.y;
      acc[0] = fma(dx, dx, fma(dy, dy, acc[0]));
      acc[1] = fma(v.x, v.x, fma(v.y, v.y, acc[1]));
      acc[2] += (isfinite(u.x) && isfinite(u.y)) ? 0.0 : 1.0;
      if (cadence) cost_terms(a.k, b, N, lo + j, u, acc[3], acc[4], acc[5]);
    }
    block_sum<6>(acc, red);  // ends on a barrier: this step's reads of sst are done
    if (threadIdx.x == 0)
      for (int q = 0; q < 6; ++q) mine[q] = acc[q];
    __syncwarp();
    if (threadIdx.x < SPC_CL) {  // lane r pushes my partials into CTA r's slot
      const unsigned dst = spc_mapa(spc_smem_u32(&gat[buf][rank][0]), (int)threadIdx.x);
      const unsigned bar = spc_mapa(spc_smem_u32(&gbar[buf]), (int)threadIdx.x);
#pragma unroll
      for (int q = 0; q < 6; q += 2)
        asm volatile(
            "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
                dst + 8 * q),
            "d"(mine[q]), "d"(mine[q + 1]), "r"(bar)
            : "memory");
    }
    if (threadIdx.x == 0) {
      asm volatile(
          "{\n.reg .pred P;\nW_%=:\n"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
          "@!P bra W_%=;\n}\n" ::"r"(spc_smem_u32(&gbar[buf])),
          "r"((unsigned)(step >> 1) & 1u)
          : "memory");
      double t[6] = {0, 0, 0, 0, 0, 0};
      for (int r = 0; r < SPC_CL; ++r)  // fixed order: the same totals in every CTA
        for (int q = 0; q < 6; ++q) t[q] += gat[buf][r][q];
      StepCtl c = a.ctl;
      c.defer_commit = cadence ? 1 : 0;
      record_step(sst, b, t[0], t[1], t[2], a.S, c, tr);
      if (cadence) {
        if (sst.k % c.log_every == 0) {
          const double inv = 1.0 / (double)N;
          const CostArgs ca = cost_view(a.H, a.W, COST_RECORD, a.sigma, a.alpha, c, tr);
          cost_finish(sst, b, t[3] * inv, t[4] * inv, t[5] * inv, a.k.rh != nullptr, ca);
        }
        commit_step(sst, c.phase);
      }
      s_copy = cadence && copy_best && sst.copy_best;
      s_go = takes_step(sst, a.ctl.phase);
    }
    __syncthreads();
    if (s_copy) {  // k_copy_view(best <- cur), my frequencies
      cd* d = reinterpret_cast<cd*>(best + (long long)b * 2 * N) + lo;
      for (int j = threadIdx.x; j < nf; j += blockDim.x) st_cd(d + j, xs[j]);
    }
  }
  cluster.sync();  // no CTA leaves while a peer's pushes may still target it
  if (rank == 0 && threadIdx.x == 0) a.st[b] = sst;
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
bool spec_steps_fits(int B, long long N) {
  static int ok = -1;
  if (ok < 0) {
    const size_t smem = (size_t)3 * SPC_MAXF * sizeof(cd);
    ok = cudaFuncSetAttribute(k_spec_steps, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem) == cudaSuccess &&
         cudaFuncSetAttribute(k_spec_steps, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
             cudaSuccess;
    if (ok) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = SPC_CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(SPC_CL, 1);
      cfg.blockDim = dim3(SPC_THREADS);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      ok = cudaOccupancyMaxActiveClusters(&nc, k_spec_steps, &cfg) == cudaSuccess && nc > 0;
    }
    cudaGetLastError();
  }
  const char* e = getenv("REDVE_SPEC_FUSED");
  if (e && e[0] == '0') return false;
  return ok == 1 && N <= (long long)SPC_CL * SPC_MAXF && (long long)B * SPC_CL <= 148;
}

int launch_spec_steps(const SpecStepArgs& a, int nsteps, unsigned cadence_mask, int copy_best,
                      double* best, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = SPC_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(SPC_CL, a.B);
  cfg.blockDim = dim3(SPC_THREADS);
  cfg.dynamicSmemBytes = (size_t)3 * SPC_MAXF * sizeof(cd);
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, k_spec_steps, a, nsteps, cadence_mask, copy_best, best);
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
