// One-kernel Fourier fixed-point step for 256 x 256 image pairs (fused.cu).
#pragma once

#include "kernels.cuh"

namespace redve {

struct FusedArgs {
  int B;
  View xin;            // x_k (ring view)
  DenoiseArgs dn;
  double* fout;        // optional [B][N] f(x_k) (cadence steps)
  const cd* tws;       // stage-major twiddles of L = 256
  const double* g;     // [H][W] spectral multiplier
  double scale;        // alpha
  View out;            // x_{k+1} (ring view)
  const double* base;  // x_b [B][N]
  View xprev;          // x_k again, for the step norm
  int S;
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  double* partials;    // [npairs][8][6]
  unsigned* counters;  // [npairs]
};

bool fused_step_ok(int H, int W, const DenoiseArgs& d);
void launch_fused_step(const FusedArgs& a, int npairs, cudaStream_t s);

}  // namespace redve
