// Slab primitives for the spatially partitioned solve (slab.cu).
#pragma once

#include "state.cuh"

namespace redve {

constexpr int SLAB_BLOCKS = 1184;  // CTA cap of the streaming reductions (8 per SM)
constexpr int GRAM_BLOCKS = 592;   // CTA cap of the window Gram (4 per SM)

void launch_vec_reduce(int op, long long n, const double* x, const double* y, double* part,
                       double* out, cudaStream_t s);  // op 0: dot, 1: squared distance
void launch_vec_axpby(long long n, double a, const double* x, double b, double* y,
                      cudaStream_t s);
void launch_halo_push(int rows, int W, int halo, const double* x, double* ext, double* prev_bot,
                      double* next_top, cudaStream_t s);
void launch_fidelity(int Hext, int W, int row0, int Hg, int h, int rows, int f,
                     const double* taps, int k, const double* x, const double* yup, double* part,
                     double* out, cudaStream_t s);
void launch_window_gram(int rows, long long n, const double* w, double* part, double* G,
                        cudaStream_t s);
void launch_window_combine(long long n, const double* w, int ke, const double* xi, double* out,
                           cudaStream_t s);

}  // namespace redve
