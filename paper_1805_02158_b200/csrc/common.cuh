// Shared device helpers for the RED / vector-extrapolation kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef REDVE_HD
#define REDVE_HD __host__ __device__ __forceinline__
#endif

namespace redve {

// ---------------------------------------------------------------- complex fp64
struct cd {
  double x, y;
};
REDVE_HD cd mk(double a, double b) { return cd{a, b}; }
REDVE_HD cd operator+(cd a, cd b) { return cd{a.x + b.x, a.y + b.y}; }
REDVE_HD cd operator-(cd a, cd b) { return cd{a.x - b.x, a.y - b.y}; }
REDVE_HD cd operator*(cd a, double s) { return cd{a.x * s, a.y * s}; }
REDVE_HD cd cmul(cd a, cd b) { return cd{fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)}; }
// multiply by conj(b)
REDVE_HD cd cmulc(cd a, cd b) { return cd{fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y)}; }

__device__ __forceinline__ cd ld_cd(const cd* p) {
  double2 v = *reinterpret_cast<const double2*>(p);
  return cd{v.x, v.y};
}
__device__ __forceinline__ void st_cd(cd* p, cd v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.x, v.y);
}
__device__ __forceinline__ cd ldg_cd(const cd* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return cd{v.x, v.y};
}

// ---------------------------------------------------------------- reductions
// Deterministic block sum of up to NV doubles per thread (fixed tree order).
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem_red /* >= 32*NV */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(0xffffffffu, v[i], o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) smem_red[i * 32 + warp] = v[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nwarps ? smem_red[i * 32 + lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      v[i] = s;
    }
  }
  __syncthreads();
}

// "Last block done" handshake: every block of a group publishes partials, then
// the block that arrives last (per group) sees all of them.  Returns true in
// the last block.  Counter is reset by the last block, so it can be reused.
// Thread 0 writes its block's partials, so thread 0 alone fences them before
// counting: the other threads' outputs (only read by later kernels) are not
// waited for -- a block-wide fence stalled every thread on its own stores.
__device__ __forceinline__ bool last_block_of_group(unsigned int* counter, unsigned int nblocks,
                                                    int* smem_flag) {
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    int last = (prev == nblocks - 1);
    if (last) *counter = 0u;
    *smem_flag = last;
  }
  __syncthreads();
  bool last = *smem_flag != 0;
  if (last) __threadfence();
  return last;
}

// Sum of the NV partials of nblk CTAs ([nblk][NV] at part) by the whole last
// CTA: lane-strided L2 loads, then the fixed block_sum tree (deterministic).
// Result valid in thread 0.
template <int NV>
__device__ __forceinline__ void gather_partials(const double* part, int nblk, double (&tot)[NV],
                                                double* smem_red /* >= 32*NV */) {
#pragma unroll
  for (int i = 0; i < NV; ++i) tot[i] = 0.0;
  for (int blk = threadIdx.x; blk < nblk; blk += blockDim.x)
#pragma unroll
    for (int i = 0; i < NV; ++i) tot[i] += __ldcg(part + (long long)blk * NV + i);
  block_sum<NV>(tot, smem_red);
}

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

}  // namespace redve
