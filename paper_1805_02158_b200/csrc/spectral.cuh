// Spectral route: the RED fixed point for LINEAR shift-invariant denoisers on
// circulant operators, iterated in the Fourier domain.
#pragma once

#include "kernels.cuh"

namespace redve {

// With f(x) = h_f * x (GaussianFilter, Identity) the fixed-point step
// (objective.py:100-104)  x+ = IDFT( DFT(H^T y / s^2 + a f(x)) / d )  is, per
// frequency k,   X+(k) = Xb(k) + m(k) X(k),   m = a hf(k) / d(k),
// with Xb = DFT(x_b) the problem's constant part.  Every quantity the drivers
// record is an inner product, so Parseval (sum |x|^2 = (1/N) sum |X|^2) gives
// them without leaving the Fourier domain:
//   step norm  ||X+ - X|| / ||X||                      (solvers.py:229-230)
//   ||Hx - y||^2 = (1/N) sum |H(k) X(k) - Y(k)|^2       (objective.py:78-81)
//   x.(x - f)   = (1/N) sum |X(k)|^2 (1 - Re hf(k))     (objective.py:83-85)
//   ||x - ref||^2 = (1/N) sum |X(k) - R(k)|^2           (imaging.py:234-248)
// and the VE Gram / recombination are inner products / linear combinations
// of the (real-viewed) spectra, equal to N times the spatial ones -- the
// rank / degeneracy decisions are scale invariant.  One DFT at the start, one
// inverse DFT at the end; every step is one pointwise kernel.
struct SpecConsts {
  const cd* m;       // [N] a hf / d
  const cd* hh;      // [N] H(k)
  const double* wr;  // [N] 1 - Re hf(k)
  const cd* xb;      // [B][N] DFT(x_b)
  const cd* yh;      // [B][N] DFT(y)
  const cd* rh;      // [B][N] DFT(ref) or null
};

struct SpecStepArgs {
  int B, H, W;
  View cur, nxt;     // spectra in the ring, viewed as doubles (2 per frequency)
  SpecConsts k;
  int cadence;       // 1: also record cost / PSNR of x+ (fused)
  double sigma, alpha;
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  int S;
  double* partials;
  unsigned* counters;
};

struct SpecCostArgs {
  int B, H, W;
  View x;
  SpecConsts k;
  int mode;          // COST_INIT / COST_FINAL
  double sigma, alpha;
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  double* partials;
  unsigned* counters;
};

int spec_chunks(int B, long long N);
void launch_spec_step(const SpecStepArgs& a, cudaStream_t s);
void launch_spec_cost(const SpecCostArgs& a, cudaStream_t s);
// The spectral schedule on chip, one cluster launch per image: steps k in
// [kstart, budget) (cadence by ctl.log_every, or every step with all_cadence),
// with the VE step (va) after each full cycle of clen steps when ve != 0;
// copy_best: cadence steps copy an improved iterate to best.  spec_run_fits
// says whether the batch / size / kappa qualify.
bool spec_run_fits(int B, long long N, int kp1);
int launch_spec_run(const SpecStepArgs& a, const VeArgs& va, int kstart, int budget, int clen,
                    int ve, int all_cadence, int copy_best, double* best, cudaStream_t s);
// real [B][N] (plain stride N) -> complex [B] at out + b*odist (imag 0), non-finite flag
void launch_spec_pack(const double* x, int B, long long N, cd* out, long long odist, int* bad,
                      cudaStream_t s);
// k x k taps (anchored at the centre, imaging.py:113-129) embedded into a zero N-image
void launch_spec_embed(const double* taps, int k, int H, int W, cd* out, cudaStream_t s);
// m = alpha hf / d with 1/d = g H W;  wr = 1 - Re hf   (hf == null: identity, hf = 1)
void launch_spec_consts(const cd* hf, const double* g, double alpha, long long N, cd* m,
                        double* wr, cudaStream_t s);
// spectrum of image b: current ring slot, or the best plain iterate if chosen
void launch_spec_pick(cd* out, View cur, const double* best, int B, long long N,
                      const ImgState* st, cudaStream_t s);
// out[b][i] = Re(z[b][i]) * scale
void launch_spec_real(const cd* z, double* out, int B, long long N, double scale, cudaStream_t s);

}  // namespace redve
