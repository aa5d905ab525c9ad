// Kernel argument blocks and launch helpers shared by kernels.cu and capi.cu.
#pragma once

#include "denoise.cuh"
#include "fft.cuh"
#include "state.cuh"
#include "ve.cuh"

namespace redve {

struct RowFwdArgs {
  int B, H, W, lpc;
  View xin;
  DenoiseArgs dn;
  cd* Z;
  const cd* tw;   // W_L^m, m < L (runtime plans)
  const cd* tws;  // stage-major table (compile-time plans), tw_stage_size(L)
  const ImgState* st;
  int phase;
  double* fout;  // optional [B][N]: f(x) as computed (cost identity on cadence steps)
};

struct ColArgs {
  int B, H, W, lpc;
  cd* Z;
  const cd* tw;   // W_L^m, m < L (runtime plans)
  const cd* tws;  // stage-major table (compile-time plans), tw_stage_size(L)
  const double* g;
  double scale;
  const ImgState* st;
  int phase;
};

struct RowInvArgs {
  int B, H, W, lpc;
  const cd* Z;
  const cd* tw;   // W_L^m, m < L (runtime plans)
  const cd* tws;  // stage-major table (compile-time plans), tw_stage_size(L)
  View out;
  const double* base;  // x_b [B][H*W] (added) or null
  View xprev;          // epilogue: previous iterate
  int epilogue;        // 1: record a fixed-point step
  int S;
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  double* partials;
  unsigned* counters;
};

enum CostMode : int { COST_RECORD = 0, COST_INIT = 1, COST_FINAL = 2, COST_VALUE = 3 };

struct CostArgs {
  int B, H, W, rows;  // rows per CTA
  int Hy, Wy, factor;
  View x;
  const double* y;
  const double* ref;
  DenoiseArgs dn;
  const double* fext;  // external f [B][N] (DN_EXTERNAL)
  const double* htaps;
  int hk;
  int separable;      // htaps == outer(hu, hv): two 1-D passes
  const double* hu;
  const double* hv;
  double sigma, alpha;
  int mode;
  double* out_vals;  // COST_VALUE: [B][3] = ||Hx-y||^2, x.(x-f), ||x-ref||^2
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  double* partials;
  unsigned* counters;
  // Fourier-route identity (cost_fp): f(x_prev) of the step, H^T y / sigma^2, ||y||^2
  const double* fprev;
  const double* hty;
  const double* yy;
};

__device__ inline double psnr_from(double ssd, long long n) {
  double mse = ssd / (double)n;
  if (mse == 0.0) return INFINITY;
  if (!isfinite(mse)) return -INFINITY;
  return 10.0 * log10(255.0 * 255.0 / mse);
}

__device__ inline void cost_finish(ImgState& s, int b, double fid, double reg, double ssd, bool has_ref,
                            const CostArgs& a) {
  const double cost = fid / (2.0 * a.sigma * a.sigma) + a.alpha * (0.5 * reg);
  const long long N = (long long)a.H * a.W;
  if (a.mode == COST_INIT) {
    if (isfinite(cost)) {
      s.best_cost = cost;
      s.copy_best = 1;
      s.has_best = 1;
    } else {
      s.copy_best = 0;
    }
    return;
  }
  if (a.mode == COST_FINAL) {
    s.use_best = (s.has_best && !(isfinite(cost) && cost <= s.best_cost)) ? 1 : 0;
    return;
  }
  const long long i = (long long)b * a.tr.cap + (s.k - 1);
  if (s.k - 1 < a.tr.cap) {
    a.tr.cost[i] = cost;
    if (has_ref) a.tr.psnr[i] = psnr_from(ssd, N);
  }
  s.copy_best = 0;
  if (a.ctl.track_best && cost < s.best_cost) {
    s.best_cost = cost;
    s.copy_best = 1;
    s.has_best = 1;
  }
  if (!isfinite(cost) && s.err == ERR_NONE) s.err = ERR_NONFINITE_COST;
}

__device__ __forceinline__ bool cost_wants(const ImgState& s, const CostArgs& a) {
  if (a.mode == COST_RECORD) return s.stepped && (s.k % a.ctl.log_every == 0);
  if (a.mode == COST_INIT || a.mode == COST_VALUE) return true;
  return s.err == ERR_NONE;  // final
}


struct VeArgs {
  int B;
  long long N;
  int m, kp1, S;
  double* ring;
  long long img_stride, slot_stride;
  ImgState* st;
  TraceBufs tr;
  double* partials;
  unsigned* counters;
  double* qscratch;  // MGS [B][kp1][N]
  int method;
  double rank_tol;
  int chunks;
  int stationary_continues;  // spectral route, tol == 0: an exactly stationary window is skipped
  int mgs_cluster;           // 1: flagged windows go to k_mgs_cluster (launched after k_gram)
};

// launchers (kernels.cu)
int configure_kernels();  // returns a cudaError_t
void launch_twiddles(cd* tw, int L, cudaStream_t s);
void launch_stage_twiddles(cd* tws, int L, cudaStream_t s);  // power-of-two L >= 16
void launch_inv_denom(double* g, int H, int W, const double* taps, int hk, double sigma,
                      double alpha, cudaStream_t s);
size_t row_fwd_smem(int W, int lpc, int radius, int ksize);
size_t col_smem(int H, int lpc);
size_t row_inv_smem(int W, int lpc);
void launch_row_fwd(const RowFwdArgs& a, int npairs, cudaStream_t s);
void launch_col(const ColArgs& a, int npairs, cudaStream_t s);
void launch_row_inv(const RowInvArgs& a, int npairs, cudaStream_t s);
int cost_rows(int H);
int cost_fp_rows(int W);
void launch_sumsq(const double* y, long long n, int B, double* out, cudaStream_t s);
void launch_cost(const CostArgs& a, int npairs, cudaStream_t s);
bool cost_fast_ok(const CostArgs& a);
void launch_cost_fast(const CostArgs& a, int npairs, cudaStream_t s);
bool cost_fp_ok(const CostArgs& a);
void launch_cost_fp(const CostArgs& a, int npairs, cudaStream_t s);
void launch_copy_view(View dst, View src, int B, long long N, const ImgState* st, int only_flag,
                      cudaStream_t s);
void launch_gram(const VeArgs& a, cudaStream_t s);
// exact MGS of the windows k_gram flagged, one 8-CTA cluster per image (no-op otherwise)
void launch_mgs_cluster(const VeArgs& a, cudaStream_t s);
bool mgs_cluster_pays(int B);
void launch_combine(const VeArgs& a, cudaStream_t s);
void launch_init_state(ImgState* st, int B, cudaStream_t s);
void launch_load_x0(double* ring, long long img_stride, const double* x0, int B, long long N,
                    int* bad, cudaStream_t s);
void launch_gather(double* out, View cur, const double* best, int B, long long N,
                   const ImgState* st, cudaStream_t s);
void launch_conv(const double* x, double* out, int B, int H, int W, const double* taps, int k,
                 int corr, double scale, cudaStream_t s);
// rank-one taps (uv = [u | v]): two 1-D passes; false if k is not compiled
bool launch_conv_rank1(const double* x, double* out, int B, int H, int W, const double* uv, int k,
                       int corr, double scale, cudaStream_t s);
void launch_decimate_conv(const double* x, double* out, int B, int H, int W, int factor,
                          const double* taps, int k, cudaStream_t s);
void launch_upsample_corr(const double* z, double* out, int B, int H, int W, int factor,
                          const double* taps, int k, double scale, cudaStream_t s);
void launch_median3(const double* x, double* out, int B, int H, int W, cudaStream_t s);
void launch_window_extrapolate_setup(ImgState* st, int B, int S, int m, cudaStream_t s);

}  // namespace redve
