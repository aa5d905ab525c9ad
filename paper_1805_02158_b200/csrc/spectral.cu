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

// The spectral route of a small batch as ONE cluster launch per image
// (configs[0]: launch-bound, ~350 tiny kernels per solve otherwise).  A
// cluster of SPC_CL CTAs holds the image's spectrum and its step constants
// (m, Xb) in shared memory, so a step costs no launch and no HBM round trip;
// every new spectrum still lands in the ring (the VE window reads it there).
//  * each step is k_spec_step's arithmetic verbatim;
//  * reductions travel by DSMEM push: every CTA st.async's its partial sums
//    into every CTA's gather slot, completing on the receiver's mbarrier (no
//    cluster barrier, hence no release fence waiting on the ring stores); all
//    CTAs then sum the slots in the same rank order, so every CTA holds the
//    same totals and applies the record / cadence cost / commit and the VE
//    decision (decide_from_gram) to its own shared copy of the image state;
//    rank 0 alone writes traces and, at the end, the state;
//  * a full cycle is followed, as in the launch schedule, by the VE step:
//    the window's Gram matrix over the cluster, the decision, the exact MGS
//    for a window the Gram route flags (cluster dot products), and the
//    recombination into the cycle-start slot, accepted only if finite.
// Reduction orders differ from the per-launch kernels (rounding-level
// differences in sums, decisions identical on the test problems).
constexpr int SPC_CL = 16, SPC_THREADS = 512, SPC_MAXF = 4096;  // frequencies per CTA
constexpr int SPC_MAXV = 22;                                     // widest pushed partial (Gram)

__device__ __forceinline__ unsigned spc_smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned spc_mapa(unsigned addr, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

struct SpcShared {
  double red[32 * SPC_MAXV];
  __align__(16) double mine[SPC_MAXV];
  __align__(16) double gat[2][SPC_CL][SPC_MAXV];  // by reduction parity, by sender rank
  __align__(16) double tot[SPC_MAXV];
  __align__(8) unsigned long long gbar[2];
  ImgState sst;  // this CTA's copy of the image state
  double R[MAXKP1][MAXKP1];
  double part[2];
  double val;
  int go, copy, acc_ok;
};

// Sum of NV doubles (thread 0's block totals in sh.mine) over the cluster, in
// rank order, into sh.tot of every CTA.  `seq` counts the calls (parity).
template <int NV>
__device__ __forceinline__ void spc_allsum(SpcShared& sh, int rank, int& seq) {
  constexpr int NV2 = (NV + 1) & ~1;  // whole 16-byte stores
  const int buf = seq & 1;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     spc_smem_u32(&sh.gbar[buf])),
                 "r"(SPC_CL * NV2 * 8)
                 : "memory");
  __syncwarp();
  if (threadIdx.x < SPC_CL) {  // lane r pushes my partials into CTA r's slot
    const unsigned dst = spc_mapa(spc_smem_u32(&sh.gat[buf][rank][0]), (int)threadIdx.x);
    const unsigned bar = spc_mapa(spc_smem_u32(&sh.gbar[buf]), (int)threadIdx.x);
#pragma unroll
    for (int q = 0; q < NV2; q += 2)
      asm volatile(
          "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(
              dst + 8 * q),
          "d"(sh.mine[q]), "d"(q + 1 < NV ? sh.mine[q + 1] : 0.0), "r"(bar)
          : "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile(
        "{\n.reg .pred P;\nW_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n"
        "@!P bra W_%=;\n}\n" ::"r"(spc_smem_u32(&sh.gbar[buf])),
        "r"((unsigned)(seq >> 1) & 1u)
        : "memory");
    for (int q = 0; q < NV; ++q) {
      double t = 0.0;
      for (int r = 0; r < SPC_CL; ++r) t += sh.gat[buf][r][q];  // fixed order
      sh.tot[q] = t;
    }
  }
  ++seq;
  __syncthreads();
}

template <int KP1>
__global__ void __launch_bounds__(SPC_THREADS) k_spec_run(SpecStepArgs a, VeArgs va, int kstart,
                                                          int budget, int clen, int ve,
                                                          int all_cadence, int copy_best,
                                                          double* best) {
  namespace cg = cooperative_groups;
  constexpr int NG = KP1 * (KP1 + 1) / 2;
  static_assert(NG <= SPC_MAXV, "Gram partials exceed the push slot");
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
  __shared__ SpcShared sh;
  ImgState& sst = sh.sst;
  if (threadIdx.x == 0) {
    sst = a.st[b];
    for (int i = 0; i < 2; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(spc_smem_u32(&sh.gbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  TraceBufs tr = a.tr;
  if (rank != 0) tr.cap = tr.ccap = 0;  // shadow records: state only, no trace writes
  auto load_cur = [&](const ImgState& s) {  // my frequencies of the current spectrum
    const cd* x = reinterpret_cast<const cd*>(a.cur.at_state(b, s)) + lo;
    for (int j = threadIdx.x; j < nf; j += blockDim.x) xs[j] = ld_cd(x + j);
  };
  load_cur(a.st[b]);
  {
    const cd* xb = a.k.xb + (long long)b * N + lo;
    for (int j = threadIdx.x; j < nf; j += blockDim.x) {
      ms[j] = ldg_cd(a.k.m + lo + j);
      bs[j] = ldg_cd(xb + j);
    }
  }
  cluster.sync();  // every CTA's mbarriers are initialised before any push
  int seq = 0;

  // ---- one fixed-point step (k_spec_step + the cadence copy_view)
  auto step = [&](bool cadence) {
    if (threadIdx.x == 0) sh.go = takes_step(sst, a.ctl.phase);
    __syncthreads();
    if (!sh.go) return;
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
    block_sum<6>(acc, sh.red);  // ends on a barrier: this step's reads of sst are done
    if (threadIdx.x == 0)
      for (int q = 0; q < 6; ++q) sh.mine[q] = acc[q];
    spc_allsum<6>(sh, rank, seq);
    if (threadIdx.x == 0) {
      const double* t = sh.tot;
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
      sh.copy = cadence && copy_best && sst.copy_best;
    }
    __syncthreads();
    if (sh.copy) {  // k_copy_view(best <- cur), my frequencies
      cd* d = reinterpret_cast<cd*>(best + (long long)b * 2 * N) + lo;
      for (int j = threadIdx.x; j < nf; j += blockDim.x) st_cd(d + j, xs[j]);
    }
  };

  // window slot j of the cycle (doubles view)
  auto slot = [&](int j) {
    return va.ring + (long long)b * va.img_stride + (long long)(j % va.S) * va.slot_stride;
  };
  const long long dlo = 2 * lo, dhi = 2 * hi;  // my range of the doubles view

  // ---- exact MGS of the window across the cluster (k_mgs_cluster), rare
  auto mgs = [&]() {
    const int n = KP1;
    const long long Nd = va.N;
    double* Q = va.qscratch + (long long)b * n * Nd;
    if (threadIdx.x < MAXKP1 * MAXKP1) (&sh.R[0][0])[threadIdx.x] = 0.0;
    int parity = 0;
    auto cdot = [&](const double* u, const double* v) -> double {
      double acc[1] = {0.0};
      for (long long p = dlo + threadIdx.x; p < dhi; p += blockDim.x) acc[0] = fma(u[p], v[p], acc[0]);
      block_sum<1>(acc, sh.red);
      if (threadIdx.x == 0) sh.part[parity] = acc[0];
      cluster.sync();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int r = 0; r < SPC_CL; ++r) t += cluster.map_shared_rank(sh.part, r)[parity];
        sh.val = t;
      }
      __syncthreads();
      parity ^= 1;
      return sh.val;
    };
    const int s0 = sst.start + va.m;
    int rank_e = n;
    double r11 = 0.0;
    bool stationary = false;
    for (int i = 0; i < n; ++i) {
      const double* xa = slot(s0 + i);
      const double* xb = slot(s0 + i + 1);
      double* qi = Q + (long long)i * Nd;
      for (long long p = dlo + threadIdx.x; p < dhi; p += blockDim.x) qi[p] = xb[p] - xa[p];
      __syncthreads();
      for (int sweep = 0; sweep < 2; ++sweep) {
        for (int j = 0; j < i; ++j) {
          const double* qj = Q + (long long)j * Nd;
          const double proj = cdot(qj, qi);
          if (threadIdx.x == 0) sh.R[j][i] += proj;
          for (long long p = dlo + threadIdx.x; p < dhi; p += blockDim.x) qi[p] -= proj * qj[p];
          __syncthreads();
        }
      }
      const double rii = sqrt(cdot(qi, qi));
      if (threadIdx.x == 0) sh.R[i][i] = rii;
      if (i == 0) {
        if (rii < 1e-300) {
          stationary = true;
          break;
        }
        r11 = rii;
      } else if (rii < va.rank_tol * r11) {
        rank_e = i;
        break;
      }
      for (long long p = dlo + threadIdx.x; p < dhi; p += blockDim.x) qi[p] /= rii;
      __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      VeOut o;
      bool finite = true;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) finite = finite && isfinite(sh.R[i][j]);
      if (stationary) o.mode = VE_CONVERGED;
      else if (!finite) o.mode = VE_SKIP;
      else decide_from_r(sh.R, n, rank_e, va.method, o);
      sst.ve_mode = o.mode;
      if (o.mode == VE_EXTRAPOLATE) {
        sst.ve_k = o.k_used;
        sst.ve_method = o.method;
        sst.ve_fallback = o.fallback;
        sst.ve_stab = o.stab;
        for (int i = 0; i <= o.k_used; ++i) {
          sst.ve_gamma[i] = o.gamma[i];
          sst.ve_c[i] = o.c[i];
          if (i < o.k_used) sst.ve_xi[i] = o.xi[i];
        }
      }
    }
    cluster.sync();  // no CTA moves on while another may still read its sh.part
  };

  // ---- the VE step after a full cycle (k_gram, k_mgs_cluster, k_combine)
  auto ve_step = [&]() {
    if (threadIdx.x == 0) sh.go = sst.term == RUNNING || sst.term == BUDGET;  // ve_participates
    __syncthreads();
    if (!sh.go) return;
    const int s0 = sst.start + va.m;
    {  // Gram of the window's differences over my range
      const double* w[KP1 + 1];
#pragma unroll
      for (int j = 0; j <= KP1; ++j) w[j] = slot(s0 + j);
      double acc[NG];
#pragma unroll
      for (int i = 0; i < NG; ++i) acc[i] = 0.0;
      for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) {
        double d0[KP1], d1[KP1];
        double2 prev = __ldcg(reinterpret_cast<const double2*>(w[0]) + p);
#pragma unroll
        for (int j = 0; j < KP1; ++j) {
          const double2 nx = __ldcg(reinterpret_cast<const double2*>(w[j + 1]) + p);
          d0[j] = nx.x - prev.x;
          d1[j] = nx.y - prev.y;
          prev = nx;
        }
        int q = 0;
#pragma unroll
        for (int i = 0; i < KP1; ++i)
#pragma unroll
          for (int j = i; j < KP1; ++j) {
            acc[q] = fma(d0[i], d0[j], acc[q]);
            acc[q] = fma(d1[i], d1[j], acc[q]);
            ++q;
          }
      }
      block_sum<NG>(acc, sh.red);
      if (threadIdx.x == 0)
        for (int q = 0; q < NG; ++q) sh.mine[q] = acc[q];
      spc_allsum<NG>(sh, rank, seq);
    }
    if (threadIdx.x == 0) {
      double G[KP1 * KP1];
      int q = 0;
      for (int i = 0; i < KP1; ++i)
        for (int j = i; j < KP1; ++j) {
          G[i * KP1 + j] = sh.tot[q];
          G[j * KP1 + i] = sh.tot[q];
          ++q;
        }
      VeOut o;
      decide_from_gram(G, KP1, va.method, va.rank_tol, o);
      sst.ve_mode = o.mode;
      if (o.mode == VE_EXTRAPOLATE) {
        sst.ve_k = o.k_used;
        sst.ve_method = o.method;
        sst.ve_fallback = o.fallback;
        sst.ve_stab = o.stab;
        for (int i = 0; i <= o.k_used; ++i) {
          sst.ve_gamma[i] = o.gamma[i];
          sst.ve_c[i] = o.c[i];
          if (i < o.k_used) sst.ve_xi[i] = o.xi[i];
        }
      }
    }
    __syncthreads();
    if (sst.ve_mode == VE_MGS) mgs();
    const int mode = sst.ve_mode;
    if (mode != VE_EXTRAPOLATE) {
      __syncthreads();
      if (threadIdx.x == 0) {
        sh.acc_ok = 0;
        if (mode == VE_CONVERGED && !va.stationary_continues) {
          sst.cur = (sst.start + va.m) % va.S;
          sst.term = CONVERGED;
          sh.acc_ok = 1;  // the current iterate moved: reload
        }
        sst.start = sst.cur;
      }
      __syncthreads();
      if (sh.acc_ok) {
        load_cur(sst);
        __syncthreads();
      }
      return;
    }
    // x = x_m + sum_{j<ke} xi_j (x_{m+j+1} - x_{m+j}) over the cycle-start slot
    const int ke = sst.ve_k;
    double xi[KP1 - 1];
#pragma unroll
    for (int j = 0; j < KP1 - 1; ++j) xi[j] = j < ke ? sst.ve_xi[j] : 0.0;
    const double* w[KP1];
#pragma unroll
    for (int j = 0; j < KP1; ++j) w[j] = slot(s0 + j);
    double* out = slot(sst.start);
    double nfv[1] = {0.0};
    for (long long p = lo + threadIdx.x; p < hi; p += blockDim.x) {
      double2 prev = __ldcg(reinterpret_cast<const double2*>(w[0]) + p);
      double2 accv = prev;
#pragma unroll
      for (int j = 0; j < KP1 - 1; ++j) {
        const double2 nx = __ldcg(reinterpret_cast<const double2*>(w[j + 1]) + p);
        accv.x = fma(xi[j], nx.x - prev.x, accv.x);
        accv.y = fma(xi[j], nx.y - prev.y, accv.y);
        prev = nx;
      }
      reinterpret_cast<double2*>(out)[p] = accv;
      nfv[0] += (isfinite(accv.x) ? 0.0 : 1.0) + (isfinite(accv.y) ? 0.0 : 1.0);
    }
    block_sum<1>(nfv, sh.red);
    if (threadIdx.x == 0) sh.mine[0] = nfv[0];
    spc_allsum<1>(sh, rank, seq);
    if (threadIdx.x == 0) {
      sh.acc_ok = sh.tot[0] == 0.0;
      if (sh.acc_ok) {
        sst.cur = sst.start;
        if (sst.k - 1 < tr.cap) tr.gamma[(long long)b * tr.cap + sst.k - 1] = sst.ve_stab;
        if (sst.ncycles < tr.ccap) {
          const long long c = (long long)b * tr.ccap + sst.ncycles;
          tr.cyc_meta[c * 4 + 0] = sst.ve_method;
          tr.cyc_meta[c * 4 + 1] = sst.ve_fallback;
          tr.cyc_meta[c * 4 + 2] = ke;
          tr.cyc_meta[c * 4 + 3] = sst.k - 1;
          tr.cyc_stab[c] = sst.ve_stab;
          for (int i = 0; i < MAXKP1; ++i) {
            tr.cyc_gamma[c * MAXKP1 + i] = i <= ke ? sst.ve_gamma[i] : 0.0;
            tr.cyc_c[c * MAXKP1 + i] = i <= ke ? sst.ve_c[i] : 0.0;
          }
        }
        sst.ncycles += 1;
      }
      sst.start = sst.cur;  // rejected: continue from the last plain iterate
    }
    __syncthreads();
    if (sh.acc_ok) {  // the extrapolated point (this CTA's own writes) is the iterate
      load_cur(sst);
      __syncthreads();
    }
  };

  // ---- the launch schedule of the solve (capi.cu device_work), on chip
  int k = kstart;
  if (!ve) {
    while (k < budget) {
      step(all_cadence || ((k + 1) % a.ctl.log_every) == 0);
      ++k;
    }
  } else {
    while (true) {
      int n = 0;
      for (int i = 0; i < clen; ++i) {
        step(((k + 1) % a.ctl.log_every) == 0);
        ++k;
        ++n;
        if (k >= budget) break;
      }
      if (n == clen) ve_step();
      if (k >= budget) break;
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
static size_t spc_dyn_smem() { return (size_t)3 * SPC_MAXF * sizeof(cd); }

template <int KP1>
static bool spc_setup() {
  static int ok = -1;
  if (ok < 0) {
    ok = cudaFuncSetAttribute(k_spec_run<KP1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)spc_dyn_smem()) == cudaSuccess &&
         cudaFuncSetAttribute(k_spec_run<KP1>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                              1) == cudaSuccess;
    if (ok) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = SPC_CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(SPC_CL, 1);
      cfg.blockDim = dim3(SPC_THREADS);
      cfg.dynamicSmemBytes = spc_dyn_smem();
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      ok = cudaOccupancyMaxActiveClusters(&nc, k_spec_run<KP1>, &cfg) == cudaSuccess && nc > 0;
    }
    cudaGetLastError();
  }
  return ok == 1;
}

static bool spc_kp1_ok(int kp1) { return kp1 >= 2 && kp1 <= 6; }

bool spec_run_fits(int B, long long N, int kp1) {
  const char* e = getenv("REDVE_SPEC_FUSED");
  if (e && e[0] == '0') return false;
  if (!spc_kp1_ok(kp1) || N > (long long)SPC_CL * SPC_MAXF || (long long)B * SPC_CL > 148)
    return false;
  switch (kp1) {
    case 2: return spc_setup<2>();
    case 3: return spc_setup<3>();
    case 4: return spc_setup<4>();
    case 5: return spc_setup<5>();
    default: return spc_setup<6>();
  }
}

template <int KP1>
static int spc_launch(const SpecStepArgs& a, const VeArgs& va, int kstart, int budget, int clen,
                      int ve, int all_cadence, int copy_best, double* best, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = SPC_CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(SPC_CL, a.B);
  cfg.blockDim = dim3(SPC_THREADS);
  cfg.dynamicSmemBytes = spc_dyn_smem();
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, k_spec_run<KP1>, a, va, kstart, budget, clen, ve,
                                 all_cadence, copy_best, best);
}

int launch_spec_run(const SpecStepArgs& a, const VeArgs& va, int kstart, int budget, int clen,
                    int ve, int all_cadence, int copy_best, double* best, cudaStream_t s) {
  switch (ve ? va.kp1 : 2) {  // the instantiation spec_run_fits prepared
    case 2: return spc_launch<2>(a, va, kstart, budget, clen, ve, all_cadence, copy_best, best, s);
    case 3: return spc_launch<3>(a, va, kstart, budget, clen, ve, all_cadence, copy_best, best, s);
    case 4: return spc_launch<4>(a, va, kstart, budget, clen, ve, all_cadence, copy_best, best, s);
    case 5: return spc_launch<5>(a, va, kstart, budget, clen, ve, all_cadence, copy_best, best, s);
    default: return spc_launch<6>(a, va, kstart, budget, clen, ve, all_cadence, copy_best, best, s);
  }
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
