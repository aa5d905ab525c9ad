// Gradient-step baselines on the device: steepest descent, SD inside VE
// cycles, and Nesterov (solvers.py:274-337; objective.py:90-93).
#pragma once

#include "state.cuh"

namespace redve {

// x_{k+1} = v - s * grad E(v),  grad E(v) = A v - H^T y / sigma^2 - alpha f(v),
// A = H^T H / sigma^2 + alpha I.
// SD:       v = x_k.
// Nesterov: v = y_k, and y_{k+1} = x_{k+1} + beta_k (x_{k+1} - x_k).
// The step norm is ||x_{k+1} - x_k|| / ||x_k|| either way (solvers.py:229-230).
struct GradArgs {
  int B, H, W;
  View v;               // where the gradient is evaluated
  View xprev;           // x_k
  View xout;            // x_{k+1}
  const double* Av;     // [B][N] A v precomputed (CG route), or null: stencil below
  const double* au;     // separable H^T H: row taps (2R+1) already scaled by 1/sigma^2
  const double* av;     //                   column taps (2R+1)
  const double* afull;  // non-separable H^T H: (2R+1)^2 taps scaled by 1/sigma^2 (au == null)
  int R;                // autocorrelation radius = ksize - 1
  const double* hty;    // [B][N] H^T y / sigma^2
  const double* f;      // [B][N] f(v)
  double alpha, step, beta;
  double* ynext;        // Nesterov: [B][N] y_{k+1}; null for SD
  double* gout;         // non-null: write grad E(v) here instead of stepping (no record)
  ImgState* st;
  StepCtl ctl;
  TraceBufs tr;
  int S;
  double* partials;
  unsigned* counters;
};

int grad_partials_per_image(int H, int W, bool stencil);
void launch_grad_step(const GradArgs& a, cudaStream_t s);

}  // namespace redve
