// Argument blocks for the super-resolution path (sr.cu).
#pragma once

#include "denoise.cuh"
#include "state.cuh"

namespace redve {

struct PwArgs {
  int B, H, W;
  int pr, sr, npos, iters;
  double inv_h2;
  View xin;          // images to denoise
  double* w0;        // [B][npos][N] raw weights of the half-plane offsets
  int w32;           // 1: w0 holds fp32 planes (specialised radii; arithmetic stays fp64)
  double* D0;        // [B][N] balancing field, ping-pong
  double* D1;
  double* out;       // [B][N] f(x)
  const ImgState* st;
  int phase;
};

enum CgMode : int { CG_INIT = 0, CG_ITER = 1, CG_RESID = 2, CG_PLAIN = 3 };

struct CgState {
  double rho, beta, alpha, atol, bn2;
  int active, its, info, zero_b, need_resid;
};

struct CgArgs {
  int B, H, W, factor, k;
  const double* taps;  // device k*k
  const double* huv;   // rank-one PSF: device [u | v] (k each), else null
  double inv_sigma2, alpha, rtol, abort;
  int maxiter;
  int row0, Hg;        // global row of local row 0 / global height (0: the buffer is the image)
  int tile_off;        // compile-time operator kernel: local row of a lattice-aligned tile origin,
  int row0m, seam;     // row0 mod Hg, local row of global row 0 (-1: none)  (set by the launcher)
  View xin;            // CG_INIT: x_k ; CG_RESID: the solution
  View xout;           // the solution being built (warm-started copy of x_k)
  const double* hty;   // [B][N] H^T y / sigma^2
  const double* f;     // [B][N] f(x_k)
  double *r, *p, *q;   // [B][N]
  CgState* cg;
  ImgState* st;
  int phase;
  double* partials;
  unsigned* counters;
};

struct RecordArgs {
  long long N;
  const CgState* cg;  // CG route: per-image iteration counts into tr.cg_iters (or null)
  View xnew, xprev;
  int S;
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  double* partials;
  unsigned* counters;
};

size_t pw_weights_smem(int pr, int sr);
void launch_pw(const PwArgs& a, cudaStream_t s, int* launches);
void launch_pw_maps(const PwArgs& a, cudaStream_t s, int* launches, double* maps);
size_t cg_matvec_smem(int k);
int cg_matvec_blocks(int H, int W);
int cg_update_blocks(long long N);
void launch_cg_init(const CgArgs& a, cudaStream_t s);
void launch_cg_iter(const CgArgs& a, cudaStream_t s);
void launch_cg_resid(const CgArgs& a, cudaStream_t s);
void launch_normal_matvec(const CgArgs& a, cudaStream_t s);  // q = A w, every row
void launch_cg_update(const CgArgs& a, cudaStream_t s);
void launch_cg_continue(const CgArgs& a, cudaGraphConditionalHandle h, cudaStream_t s);
void launch_cg_zero_b(const CgArgs& a, cudaStream_t s);
void launch_step_record(const RecordArgs& a, int B, cudaStream_t s);
void launch_denoise_view(View xin, DenoiseArgs dn, double* out, const ImgState* st, int phase,
                         int B, int H, int W, cudaStream_t s);

}  // namespace redve
