// Filter-bank (reaction-diffusion) denoiser arguments (rd.cu).
#pragma once

#include "state.cuh"

namespace redve {

struct RdArgs {
  int B, H, W;
  int nf, fs;
  const double* filters;  // device [nf][fs][fs]
  const double* scales;   // device [nf]
  double tau;
  View xin;
  double* out;            // [B][N]
  const ImgState* st;
  int phase;
};

size_t rd_smem(int nf, int fs);
void launch_rd(const RdArgs& a, cudaStream_t s);

}  // namespace redve
